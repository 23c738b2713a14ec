#!/bin/bash
# abx.sh V... : per variant lib: quick parity (C2-shape S/PCG vs port), per-pass burst times and the
# in-chain per-iteration slope (SHAPE env: "nt n1 n2", default C2).  Interleave base/variant for A/B.
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  par=$(FDG_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "pcg_noncube or precond_noncube" 2>&1 | tail -1)
  pt=$(FDG_LIB=$lib timeout 120 python scripts/pass_times.py 2>&1 | tail -1)
  sl=$(FDG_LIB=$lib timeout 300 python scripts/iter_slope.py $SHAPE 2>&1 | tail -2 | tr '\n' ' ')
  echo "$v | $par | $pt | $sl"
done
