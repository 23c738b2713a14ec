# r2_exp9.sh : TMA staging of the Hartley row passes / Q-split rows; per-row bulk copies of the column P passes (A/B)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp9_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -1 gpurun_out/exp9_tests.log
[ $rc -eq 0 ] || exit 1
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_pcol.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "precond" > gpurun_out/exp9_tests_pcol.log 2>&1; echo pcol_tests_rc=$?; tail -1 gpurun_out/exp9_tests_pcol.log
bash scripts/abx.sh base notmap pcol base 2>&1 | tee gpurun_out/exp9_c2.txt
SHAPE="128 512 512" bash scripts/abx.sh base notmap pcol 2>&1 | tee gpurun_out/exp9_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base notmap 2>&1 | tee gpurun_out/exp9_c4.txt
