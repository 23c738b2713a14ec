# r2_exp28.sh : Hartley row pass with the r.z dot: L2 prefetch of the dot operand at the tile start (base) vs rp0
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp28_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -2 gpurun_out/exp28_tests.log
[ $rc -eq 0 ] || exit 1
bash scripts/abx.sh rp0 base rp0 base 2>&1 | tee gpurun_out/exp28_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh rp0 base 2>&1 | tee gpurun_out/exp28_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh rp0 base 2>&1 | tee gpurun_out/exp28_c4.txt
