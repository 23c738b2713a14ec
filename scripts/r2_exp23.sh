# r2_exp23.sh : K2 per-slice scalars requested before the tile wait + row fold in the G = 4 split-interleaved exchange slots (base) vs head
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp23_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp23_tests.log
[ $rc -eq 0 ] || exit 1
SHAPE="128 1024 1024" bash scripts/abx.sh head base head base 2>&1 | tee gpurun_out/exp23_c4.txt
SHAPE="128 512 512" bash scripts/abx.sh head base head base 2>&1 | tee gpurun_out/exp23_c3.txt
bash scripts/abx.sh head base head base 2>&1 | tee gpurun_out/exp23_c2.txt
