# r2_exp5.sh : L2 prefetch of the next tile in the unstaged passes (C1 matvec, C4 1024-point Hartley, C2 check)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c1.py -q -m gpu -x > gpurun_out/exp5_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/exp5_tests.log
for v in base nopf base nopf; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "$v | $(FDG_LIB=$lib timeout 300 python scripts/bench_c1.py 2>&1 | tail -1)"
done 2>&1 | tee gpurun_out/exp5_c1.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base nopf base 2>&1 | tee gpurun_out/exp5_c4.txt
bash scripts/abx.sh base nopf 2>&1 | tee gpurun_out/exp5_c2.txt
