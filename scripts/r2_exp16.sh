# r2_exp16.sh : Q-split trivial factors (base vs qt0); lane-major column exchanges at L = 1024 (ly1k) and L = 2048 (ly2k)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_solves.py -q -m gpu -x > gpurun_out/exp16_tests.log 2>&1; rc=$?; echo tests_rc=$rc; tail -3 gpurun_out/exp16_tests.log
[ $rc -eq 0 ] || exit 1
for v in ly1k ly2k; do FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp16_tests_$v.log 2>&1; echo ${v}_tests_rc=$?; tail -1 gpurun_out/exp16_tests_$v.log; done
SHAPE="128 512 512" bash scripts/abx.sh qt0 base ly1k qt0 base ly1k 2>&1 | tee gpurun_out/exp16_c3.txt
SHAPE="128 1024 1024" bash scripts/abx.sh base ly2k base ly2k 2>&1 | tee gpurun_out/exp16_c4.txt
