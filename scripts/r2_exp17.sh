# r2_exp17.sh : L = 1024 split column pass as two 128-thread CTAs per SM (twist by constants frees the table's 8 KB): c128; twist table off alone: tws256
mkdir -p gpurun_out
for v in c128; do FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/exp17_tests_$v.log 2>&1; echo ${v}_tests_rc=$?; tail -1 gpurun_out/exp17_tests_$v.log; done
SHAPE="128 512 512" bash scripts/abx.sh base c128 tws256 base c128 tws256 2>&1 | tee gpurun_out/exp17_c3.txt
