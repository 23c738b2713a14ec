# r2_src_c4all.sh : source-level ncu (stall samples + bank conflicts by line) of every kernel of one C4 / C3 iteration
mkdir -p gpurun_out /tmp/reps
for cfg in C4 C3; do
CONFIG=$cfg MAXIT=1 ncu -f --set full --import-source on --clock-control none \
  -k regex:"k_row|k_col|k_hartley|k_t_filter" -s 7 -c 8 -o /tmp/reps/srcfull_$cfg \
  python scripts/prof_c2.py > gpurun_out/ncu_srcfull_$cfg.log 2>&1; echo srcfull_$cfg=$?
ncu -i /tmp/reps/srcfull_$cfg.ncu-rep --page source --csv --print-source cuda,sass > /tmp/reps/srcfull_$cfg.csv 2>&1
python scripts/src_conflicts.py /tmp/reps/srcfull_$cfg.csv 8 > gpurun_out/conflicts_$cfg.txt 2>&1
for k in "k_rowc<(int)2048, (int)2" "k_rowc<(int)2048, (int)1" "k_rowq<(int)1024, (int)2" "k_rowq<(int)1024, (int)1" "k_colc" "k_t_filter" "k_hartley_row" "k_hartley_col"; do
  python scripts/src_hot.py /tmp/reps/srcfull_$cfg.csv "$k" 14
done > gpurun_out/hot_$cfg.txt 2>&1
cat gpurun_out/conflicts_$cfg.txt
done
