# r2_exp13.sh : twist factors by constants (base: M = 1024 only; tc0: tables; tc2: every length); 512-thread 1024-point passes (h512)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp13_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp13_tests.log
for v in tc2 h512; do FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp13_tests_$v.log 2>&1; echo ${v}_tests_rc=$?; tail -1 gpurun_out/exp13_tests_$v.log; done
SHAPE="128 1024 1024" bash scripts/abx.sh tc0 base h512 tc0 base h512 2>&1 | tee gpurun_out/exp13_c4.txt
SHAPE="128 512 512" bash scripts/abx.sh tc0 tc2 tc0 tc2 2>&1 | tee gpurun_out/exp13_c3.txt
bash scripts/abx.sh tc0 tc2 tc0 tc2 2>&1 | tee gpurun_out/exp13_c2.txt
