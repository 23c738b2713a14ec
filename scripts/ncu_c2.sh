MAXIT=2 python scripts/prof_c2.py > gpurun_out/prof_plain.log 2>&1 && \
MAXIT=2 ncu --set full --clock-control none --import-source on -k regex:"k_row|k_col|k_hartley|k_t_filter|k_cg" -c 16 -o gpurun_out/prof_c2c python scripts/prof_c2.py > gpurun_out/ncu_c2.log 2>&1
echo ncu_rc=$?
