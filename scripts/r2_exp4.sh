# r2_exp4.sh : ragged staged split rows (C1 matvec) + PFA mirror pairs: parity and timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c1.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp4_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/exp4_tests.log
for v in base norag base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  b=$(FDG_LIB=$lib timeout 300 python scripts/bench_c1.py 2>&1 | tail -1)
  echo "$v | $b"
done 2>&1 | tee gpurun_out/exp4_c1.txt
bash scripts/abx.sh base norag 2>&1 | tee gpurun_out/exp4_c2.txt
