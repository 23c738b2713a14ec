# r2_final.sh : full GPU tests + smoke + bench (both arms), then the ncu launch lists / full captures / summaries of the final kernels
mkdir -p gpurun_out
bash scripts/r2_tests.sh
bash scripts/r2_bench.sh
bash scripts/r2_prof3.sh > gpurun_out/prof3.log 2>&1; tail -3 gpurun_out/prof3.log
