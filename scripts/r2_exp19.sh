# r2_exp19.sh : C1 matvec: ragged row tiles staged flat (base) vs the unstaged direct row pass (rg0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_c1.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp19_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp19_tests.log
[ $rc -eq 0 ] || exit 1
for v in rg0 base rg0 base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  echo "$v: $(FDG_LIB=$lib python scripts/bench_c1.py 5 2>&1 | tail -1 | cut -c1-330)"
done 2>&1 | tee gpurun_out/exp19_c1.txt
