# r2_exp12.sh : radix-32 1024-point halves of the L = 2048 split passes (base) vs radix 16 (r16) vs lane-major columns (ly1)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c1.py -q -m gpu -x > gpurun_out/exp12_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp12_tests.log
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_ly1.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp12_tests_ly1.log 2>&1; echo ly1_tests_rc=$?; tail -1 gpurun_out/exp12_tests_ly1.log
SHAPE="128 1024 1024" bash scripts/abx.sh r16 base ly1 r16 base ly1 2>&1 | tee gpurun_out/exp12_c4.txt
