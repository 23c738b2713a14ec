# r2_exp22.sh : Q-split passes: symbol table de-interleaved by residue (qw0 vs head), twist from a per-thread value + staged W_64 table (base vs qw0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp22_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp22_tests.log
[ $rc -eq 0 ] || exit 1
SHAPE="128 512 512" bash scripts/abx.sh head qw0 base head qw0 base 2>&1 | tee gpurun_out/exp22_c3.txt
