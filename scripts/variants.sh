#!/bin/bash
# variants.sh V1 V2 ... : parity subset + bench (pass profile) per lib/libfdg_V.so
# ("base" = lib/libfdg.so).  Results in gpurun_out/var_V.{json,log}.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  FDG_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/var_$v.log 2>&1
  echo "$v tests: $(tail -1 gpurun_out/var_$v.log)"
  FDG_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --admm-steps 0 > gpurun_out/var_$v.json 2>>gpurun_out/var_$v.log
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/var_{v}.json"))
ps = " ".join(f"{k.split('_')[0]}={p['ms']*1e3:.0f}" for k, p in d["passes"].items())
print(f"{v}: {d['value']:.1f} it/s  {ps}")
PY
done
