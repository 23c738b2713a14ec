# shape_bench.sh V... : C1 microbenchmark + PCG pass times at the C2/C3/C4 shapes per variant library
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "== $v"
  FDG_LIB=$lib python scripts/bench_c1.py 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 matvec %.2f ms precond %.2f ms' % (d['matvec_ms'], d['precond_ms']))"
  for s in "128 512 512" "128 1024 1024"; do
    FDG_LIB=$lib timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --admm-steps 0 --shape $s > gpurun_out/sb.json 2>gpurun_out/sb.err
    python - "$s" <<'PY' || tail -3 gpurun_out/sb.err
import json, sys
d = json.load(open("gpurun_out/sb.json"))
print(sys.argv[1], round(d["value"], 1), " ".join(f"{k.split('_')[0]}={p['ms']*1e3:.0f}" for k, p in d["passes"].items()))
PY
  done
done
