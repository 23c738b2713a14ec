# r2_src_c1.sh : source-level ncu of the C1 matvec passes (direct 2048-point row / column kernels)
mkdir -p gpurun_out /tmp/reps
ncu -f --set full --import-source on --clock-control none -k regex:"k_row|k_col" -c 2 -o /tmp/reps/srcfull_C1 \
  python scripts/prof_c1.py > gpurun_out/ncu_srcfull_C1.log 2>&1; echo srcfull_C1=$?
ncu -i /tmp/reps/srcfull_C1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/reps/srcfull_C1.csv 2>&1
for k in "k_row<" "k_col<"; do python scripts/src_hot.py /tmp/reps/srcfull_C1.csv "$k" 18; done > gpurun_out/hot_C1.txt 2>&1
