# r2_exp24.sh : real symbol de-interleaved into even | odd halves (row-pass bank conflicts), unswizzled slots for the mirror exchanges (base) vs head
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py tests/test_gpu_c1.py -q -m gpu -x > gpurun_out/exp24_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp24_tests.log
[ $rc -eq 0 ] || exit 1
bash scripts/abx.sh head base head base 2>&1 | tee gpurun_out/exp24_c2.txt
SHAPE="128 1024 1024" bash scripts/abx.sh head base head base 2>&1 | tee gpurun_out/exp24_c4.txt
SHAPE="128 512 512" bash scripts/abx.sh head base 2>&1 | tee gpurun_out/exp24_c3.txt
