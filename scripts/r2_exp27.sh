# r2_exp27.sh : C1 matvec: 2048-point twiddle table in shared memory (np vs ts1), L2 prefetch of the column pass's accumulate operand (base vs np)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_c1.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp27_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp27_tests.log
[ $rc -eq 0 ] || exit 1
for v in np base np base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "$v: $(FDG_LIB=$lib python scripts/bench_c1.py 5 2>&1 | tail -1 | cut -c80-250)"
done 2>&1 | tee gpurun_out/exp27_c1.txt
