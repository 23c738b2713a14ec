# r2_exp15.sh : K2 second-convolution input from the owned registers (base) vs all from the exchange (wo0); last-pass twiddles by constants (base) vs table loads (lc0); twist constants pre-only (tcp) / combine-only (tcc)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c1.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp15_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp15_tests.log
[ $rc -eq 0 ] || exit 1
bash scripts/abx.sh wo0 base wo0 base 2>&1 | tee gpurun_out/exp15_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh lc0 base wo0 lc0 base wo0 2>&1 | tee gpurun_out/exp15_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh lc0 base tcp tcc lc0 base tcp tcc 2>&1 | tee gpurun_out/exp15_c4.txt
python scripts/bench_c1.py 3 2>&1 | tail -1 | cut -c1-400
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_lc0.so python scripts/bench_c1.py 3 2>&1 | tail -1 | cut -c1-400
