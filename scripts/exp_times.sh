# per-pass times of (possibly numerically invalid) experimental variants
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "$v $(FDG_LIB=$lib timeout 300 python scripts/pass_times.py 10 2>&1 | tail -1)"
done
