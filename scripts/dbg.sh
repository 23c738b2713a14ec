for v in s2 s3; do
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pcg_noncube" 2>&1 | grep -E "assert|Error|passed|failed" | head -20
done
