# r2_exp2.sh : PFA lanes-per-CTA variants (C1 solve time + parity) and staged 1024-point Hartley passes at C4 shape
mkdir -p gpurun_out
for v in base g3 g2c4 g3c7 base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  par=$(FDG_LIB=$lib timeout 300 python -m pytest tests/test_gpu_c1.py -q -m gpu -x -k "precond" 2>&1 | tail -1)
  b=$(FDG_LIB=$lib timeout 300 python scripts/bench_c1.py 2>&1 | tail -1)
  echo "$v | $par | $b"
done 2>&1 | tee gpurun_out/exp2_pfa.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base pf1024 base pf1024 2>&1 | tee gpurun_out/exp2_pf1024.txt
