for v in mb2 mb3; do
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so python bench.py --steps 5 --warmup 2 --no-cpu-baseline --admm-steps 0 > gpurun_out/bench_$v.json 2>gpurun_out/bench_$v.err
FDG_LIB=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
done
