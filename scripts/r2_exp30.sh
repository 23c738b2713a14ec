# r2_exp30.sh : prime-factor passes: DFT_31 with compile-time output index (constant-bank FMA operands), division-free copy loops of the column pass (base) vs head
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_c1.py -q -m gpu -x > gpurun_out/exp30_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -2 gpurun_out/exp30_tests.log
[ $rc -eq 0 ] || exit 1
for v in head base head base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "$v: $(FDG_LIB=$lib python scripts/bench_c1.py 5 2>&1 | tail -1 | cut -c80-250)"
done 2>&1 | tee gpurun_out/exp30_c1.txt
