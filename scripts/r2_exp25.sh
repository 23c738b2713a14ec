# r2_exp25.sh : t filter: the spatial eigenvalue loads requested before the wait on the staged tile (base) vs head
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp25_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp25_tests.log
[ $rc -eq 0 ] || exit 1
bash scripts/abx.sh head base head base 2>&1 | tee gpurun_out/exp25_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh head base 2>&1 | tee gpurun_out/exp25_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh head base 2>&1 | tee gpurun_out/exp25_c4.txt
