# r2_exp14.sh : t filter as complex FFT + one mirror exchange + inverse FFT (base) vs two Hartley transforms (tf0); CTA skew in K2 (sk500, sk2000)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py tests/test_gpu_c0_solve.py -q -m gpu -x > gpurun_out/exp14_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp14_tests.log
bash scripts/abx.sh tf0 base sk500 sk2000 tf0 base sk500 sk2000 2>&1 | tee gpurun_out/exp14_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh tf0 base tf0 base 2>&1 | tee gpurun_out/exp14_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh tf0 base 2>&1 | tee gpurun_out/exp14_c4.txt
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_h512.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "precond" > gpurun_out/exp14_tests_h512.log 2>&1; rc=$?; echo h512_tests_rc=$rc; tail -2 gpurun_out/exp14_tests_h512.log
[ $rc -eq 0 ] && SHAPE="128 1024 1024" bash scripts/abx.sh h512 base 2>&1 | tee gpurun_out/exp14_c4_h512.txt
