# r2_exp18.sh : Q-split row passes: own combination term from registers + MODE 2 direction update as a flat pre-pass (base) vs before (qp0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp18_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp18_tests.log
[ $rc -eq 0 ] || exit 1
SHAPE="128 512 512" bash scripts/abx.sh qp0 base qp0 base 2>&1 | tee gpurun_out/exp18_c3.txt
