# r2_src_c2.sh : source-level ncu of the C2 K passes (K1, K2, K3), exported on the box
mkdir -p gpurun_out /tmp/reps
MAXIT=1 python scripts/prof_c2.py > gpurun_out/prof_plain.log 2>&1 || { echo plain_failed; exit 1; }
MAXIT=1 ncu --set full --import-source on --clock-control none -k regex:"k_rowc|k_colc" -s 3 -c 3 -o /tmp/reps/src_c2 \
  python scripts/prof_c2.py > gpurun_out/ncu_src_c2.log 2>&1; echo src_rc=$?
ncu -i /tmp/reps/src_c2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_c2_k.csv 2>&1
ncu -i /tmp/reps/src_c2.ncu-rep --page raw --csv > gpurun_out/raw_c2_k.csv 2>&1
ls -la gpurun_out
