# r2_exp10.sh : 2-D tensor-map TMA staging of the split column passes (A/B vs per-thread cp.async)
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp10_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp10_tests.log
[ $rc -eq 0 ] || exit 1
timeout 600 python -m pytest tests/test_gpu_full_solves.py tests/test_gpu_c0_solve.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/exp10_tests2.log 2>&1; echo tests2_rc=$?; tail -1 gpurun_out/exp10_tests2.log
bash scripts/abx.sh base cols0 base cols0 2>&1 | tee gpurun_out/exp10_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh base cols0 2>&1 | tee gpurun_out/exp10_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base cols0 2>&1 | tee gpurun_out/exp10_c4.txt
