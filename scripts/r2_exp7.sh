# r2_exp7.sh : TMA (bulk copy + mbarrier) staging of the split row passes: parity first (bounded), then A/B
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp7_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -2 gpurun_out/exp7_tests.log
[ $rc -eq 0 ] || exit 1
timeout 600 python -m pytest tests/test_gpu_full_solves.py tests/test_gpu_c0_solve.py -q -m gpu -x > gpurun_out/exp7_tests2.log 2>&1; echo tests2_rc=$?; tail -1 gpurun_out/exp7_tests2.log
bash scripts/abx.sh base notma base notma 2>&1 | tee gpurun_out/exp7_c2.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base notma 2>&1 | tee gpurun_out/exp7_c4.txt
