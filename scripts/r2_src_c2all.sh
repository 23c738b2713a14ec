# r2_src_c2all.sh : source-level ncu (stall samples + bank conflicts by line) of every kernel of one C2 iteration
mkdir -p gpurun_out /tmp/reps
CONFIG=C2 MAXIT=1 ncu -f --set full --import-source on --clock-control none \
  -k regex:"k_row|k_col|k_hartley|k_t_filter" -s 7 -c 8 -o /tmp/reps/srcfull_C2 \
  python scripts/prof_c2.py > gpurun_out/ncu_srcfull_C2.log 2>&1; echo srcfull_C2=$?
ncu -i /tmp/reps/srcfull_C2.ncu-rep --page source --csv --print-source cuda,sass > /tmp/reps/srcfull_C2.csv 2>&1
python scripts/src_conflicts.py /tmp/reps/srcfull_C2.csv 8 > gpurun_out/conflicts_C2.txt 2>&1
for k in "k_rowc<(int)512, (int)2" "k_rowc<(int)512, (int)1" "k_t_filter" "k_hartley_row" "k_hartley_col"; do
  python scripts/src_hot.py /tmp/reps/srcfull_C2.csv "$k" 16
done > gpurun_out/hot_C2.txt 2>&1
cat gpurun_out/conflicts_C2.txt
