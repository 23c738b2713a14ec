#!/bin/bash
# ab.sh V... : in-chain per-iteration cost (scripts/iter_slope.py) per variant library at C2
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "$v: $(FDG_LIB=$lib timeout 300 python scripts/iter_slope.py $SHAPE 2>&1 | tail -2 | tr '\n' ' ')"
done
