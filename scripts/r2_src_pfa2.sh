# r2_src_pfa2.sh : source-level ncu of the C1 prime-factor passes
mkdir -p gpurun_out /tmp/reps
ncu -f --set full --import-source on --clock-control none -k regex:"k_pfa" -c 2 -o /tmp/reps/srcfull_pfa \
  python scripts/prof_c1.py > gpurun_out/ncu_srcfull_pfa.log 2>&1; echo srcfull_pfa=$?
ncu -i /tmp/reps/srcfull_pfa.ncu-rep --page source --csv --print-source cuda,sass > /tmp/reps/srcfull_pfa.csv 2>&1
for k in "k_pfa_hrow" "k_pfa_hcol"; do python scripts/src_hot.py /tmp/reps/srcfull_pfa.csv "$k" 16; done > gpurun_out/hot_pfa.txt 2>&1
