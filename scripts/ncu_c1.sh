# ncu_c1.sh : launch list and full capture of the C1 matvec + 2-level solve kernels
python scripts/prof_c1.py > gpurun_out/prof_c1_plain.log 2>&1 || { echo plain_failed; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C1.csv \
  python scripts/prof_c1.py > gpurun_out/ncu_ll_C1.log 2>&1
echo ll_rc=$?
ncu --set full --import-source on --clock-control none -k regex:"k_row|k_col|k_pfa|k_bs" -o gpurun_out/full_C1 \
  python scripts/prof_c1.py > gpurun_out/ncu_full_C1.log 2>&1
echo full_rc=$?
