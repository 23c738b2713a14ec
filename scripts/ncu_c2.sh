MAXIT=1 python scripts/prof_c2.py > gpurun_out/prof_plain.log 2>&1 && \
MAXIT=1 ncu --set full --clock-control none -k regex:"k_row|k_col|k_hartley|k_t_filter" -s 7 -c 8 -o gpurun_out/prof_c2d python scripts/prof_c2.py > gpurun_out/ncu_c2.log 2>&1
echo ncu_rc=$?
