# r2_exp29.sh : K2 per-slice scalars requested a whole tile ahead (base) vs at the tile start (head)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp29_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -2 gpurun_out/exp29_tests.log
[ $rc -eq 0 ] || exit 1
bash scripts/abx.sh head base head base 2>&1 | tee gpurun_out/exp29_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh head base 2>&1 | tee gpurun_out/exp29_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh head base 2>&1 | tee gpurun_out/exp29_c4.txt
