# r2_exp21.sh : Q-split output combination with a shuffle first stage (base) vs all through shared memory (qs0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp21_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp21_tests.log
[ $rc -eq 0 ] || exit 1
SHAPE="128 512 512" bash scripts/abx.sh qs0 base qs0 base 2>&1 | tee gpurun_out/exp21_c3.txt
