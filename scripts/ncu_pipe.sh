# full ncu capture of the fused preconditioner kernels (one PCG iteration) -> gpurun_out/$1.ncu-rep
name=${1:-prof_pipe}
MAXIT=1 python scripts/prof_c2.py > gpurun_out/prof_plain.log 2>&1 && \
MAXIT=1 ncu --set full --import-source on --clock-control none -k regex:"k_pc_pipe|k_t_filter" -s 3 -c 3 -o gpurun_out/$name \
  python scripts/prof_c2.py > gpurun_out/ncu_$name.log 2>&1
echo ncu_rc=$?
