timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/tests_q.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/tests_q.log
python bench.py --steps 5 --warmup 2 --no-cpu-baseline --admm-steps 0 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; echo bench_rc=$?
