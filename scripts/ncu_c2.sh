# ncu_c2.sh [name] : full ncu capture of one C2 PCG iteration's kernels -> gpurun_out/<name>.ncu-rep
# (the plain command runs first and must exit 0; never a bench number under ncu)
name=${1:-prof_c2}
MAXIT=1 python scripts/prof_c2.py > gpurun_out/prof_plain.log 2>&1 && \
MAXIT=1 ncu --set full --import-source on --clock-control none \
  -k regex:"k_row|k_col|k_hartley|k_t_filter|k_axpy_dev" -s 7 -c 9 -o gpurun_out/$name \
  python scripts/prof_c2.py > gpurun_out/ncu_$name.log 2>&1
echo ncu_rc=$?
