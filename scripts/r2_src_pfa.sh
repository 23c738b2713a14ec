# r2_src_pfa.sh : source-level ncu of the prime-factor passes (C1 solve), exported on the box
mkdir -p gpurun_out /tmp/reps
python scripts/prof_c1.py > gpurun_out/prof_c1_plain.log 2>&1 || { echo plain_failed; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"k_pfa" -c 2 -o /tmp/reps/src_pfa \
  python scripts/prof_c1.py > gpurun_out/ncu_src_pfa.log 2>&1; echo src_rc=$?
ncu -i /tmp/reps/src_pfa.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_pfa.csv 2>&1
ncu -i /tmp/reps/src_pfa.ncu-rep --page raw --csv > gpurun_out/raw_pfa.csv 2>&1
ls -la gpurun_out
