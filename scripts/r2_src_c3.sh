# r2_src_c3.sh : source-level ncu of the C3 K passes (k_rowq MODE 1 / 2, k_colc<1024,2>) and the C4 K2 / P2, exported on the box
mkdir -p gpurun_out /tmp/reps
CONFIG=C3 MAXIT=1 python scripts/prof_c2.py > gpurun_out/prof_plain_c3.log 2>&1 || { echo plain_failed; exit 1; }
CONFIG=C3 MAXIT=1 ncu --set full --import-source on --clock-control none -k regex:"k_rowq|k_colc" -s 3 -c 3 -o /tmp/reps/src_c3 \
  python scripts/prof_c2.py > gpurun_out/ncu_src_c3.log 2>&1; echo src_c3_rc=$?
ncu -i /tmp/reps/src_c3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_c3_k.csv 2>&1
CONFIG=C4 MAXIT=1 ncu --set full --import-source on --clock-control none -k regex:"k_colc|k_hartley_col" -s 2 -c 2 -o /tmp/reps/src_c4 \
  python scripts/prof_c2.py > gpurun_out/ncu_src_c4.log 2>&1; echo src_c4_rc=$?
ncu -i /tmp/reps/src_c4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_c4_k.csv 2>&1
ls -la gpurun_out | tail -5
