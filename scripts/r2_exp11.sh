# r2_exp11.sh : tensor-map TMA staging of the Hartley column / t passes; staged 1024-point Hartley passes (C4)
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp11_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp11_tests.log
[ $rc -eq 0 ] || exit 1
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_pf1024.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp11_tests_pf.log 2>&1; echo pf_tests_rc=$?; tail -1 gpurun_out/exp11_tests_pf.log
bash scripts/abx.sh base pcol0 base pcol0 2>&1 | tee gpurun_out/exp11_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh base pcol0 2>&1 | tee gpurun_out/exp11_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base pcol0 pf1024 2>&1 | tee gpurun_out/exp11_c4.txt
