python scripts/prof_c2.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_row|k_col" -s 3 -c 3 -o gpurun_out/prof_c2b python scripts/prof_c2.py > gpurun_out/ncu_c2.log 2>&1
echo ncu_rc=$?
tail -2 gpurun_out/ncu_c2.log
