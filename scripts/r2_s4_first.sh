# r2_s4_first.sh : full GPU tests + smoke + bench (both arms) of the current tree
mkdir -p gpurun_out
bash scripts/r2_tests.sh
bash scripts/r2_bench.sh
