# r2_exp1.sh : C1 PFA preconditioner parity + timing; K2 lean variants A/B at C2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c1.py -q -m gpu -x > gpurun_out/exp1_c1tests.log 2>&1; echo c1tests_rc=$?
tail -3 gpurun_out/exp1_c1tests.log
timeout 300 python scripts/bench_c1.py > gpurun_out/exp1_c1bench.json 2>&1; echo c1bench_rc=$?
cat gpurun_out/exp1_c1bench.json | tail -2
bash scripts/abx.sh base lean1 lean2 lean2m2 base lean2 2>&1 | tee gpurun_out/exp1_ab.txt
