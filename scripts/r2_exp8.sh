# r2_exp8.sh : TMA staging of the split column passes (K2) + PFA rows TMA / batched lambda loads
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp8_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -2 gpurun_out/exp8_tests.log
[ $rc -eq 0 ] || exit 1
timeout 600 python -m pytest tests/test_gpu_full_solves.py tests/test_gpu_c0_solve.py tests/test_gpu_c1.py -q -m gpu -x > gpurun_out/exp8_tests2.log 2>&1; echo tests2_rc=$?; tail -1 gpurun_out/exp8_tests2.log
bash scripts/abx.sh base nocol base nocol 2>&1 | tee gpurun_out/exp8_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh base nocol 2>&1 | tee gpurun_out/exp8_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base nocol 2>&1 | tee gpurun_out/exp8_c4.txt
for v in base nopfatma base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "$v | $(FDG_LIB=$lib timeout 300 python scripts/bench_c1.py 2>&1 | tail -1)"
done 2>&1 | tee gpurun_out/exp8_c1.txt
