# r2_exp6.sh : K2 energy from registers (A/B) + source-level ncu of the C2 K passes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp6_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/exp6_tests.log
bash scripts/abx.sh base ereg0 base ereg0 2>&1 | tee gpurun_out/exp6_c2.txt
bash scripts/r2_src_c2.sh
