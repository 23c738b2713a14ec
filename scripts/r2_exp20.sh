# r2_exp20.sh : radix-8 1024-point Hartley / direct passes at 3 (r8m3) / 4 (r8m4) CTAs per SM, and 512-thread CTAs at 64 registers (r8w)
mkdir -p gpurun_out
for v in r8m3 r8m4 r8w; do FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp20_tests_$v.log 2>&1; echo ${v}_tests_rc=$?; tail -1 gpurun_out/exp20_tests_$v.log; done
SHAPE="128 1024 1024" bash scripts/abx.sh base r8m3 r8m4 r8w base r8m3 r8m4 r8w 2>&1 | tee gpurun_out/exp20_c4.txt
