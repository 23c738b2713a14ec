# r2_exp26.sh : 1024-point Hartley passes at 3 CTAs per SM (80 registers, ~350 B of spills): m3 vs base
mkdir -p gpurun_out
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_m3.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "precond" > gpurun_out/exp26_tests_m3.log 2>&1; rc=$?; echo m3_tests_rc=$rc; tail -3 gpurun_out/exp26_tests_m3.log
[ $rc -eq 0 ] || exit 0
SHAPE="128 1024 1024" bash scripts/abx.sh base m3 base m3 2>&1 | tee gpurun_out/exp26_c4.txt
