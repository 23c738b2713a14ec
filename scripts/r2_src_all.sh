# r2_src_all.sh : source-level ncu (bank conflicts by line) of every kernel of one C2 / C4 iteration and of the C1 passes
mkdir -p gpurun_out /tmp/reps
for cfg in ${CFGS:-C2 C3 C4}; do
  CONFIG=$cfg MAXIT=1 ncu --section SourceCounters --section MemoryWorkloadAnalysis --import-source on --clock-control none \
    -k regex:"k_row|k_col|k_hartley|k_t_filter" -s 7 -c 8 -o /tmp/reps/srcall_$cfg \
    python scripts/prof_c2.py > gpurun_out/ncu_srcall_$cfg.log 2>&1; echo srcall_$cfg=$?
  ncu -i /tmp/reps/srcall_$cfg.ncu-rep --page source --csv --print-source cuda,sass > /tmp/reps/srcall_$cfg.csv 2>&1
  python scripts/src_conflicts.py /tmp/reps/srcall_$cfg.csv 8 > gpurun_out/conflicts_$cfg.txt 2>&1
done
ncu --section SourceCounters --section MemoryWorkloadAnalysis --import-source on --clock-control none -k regex:"k_pfa" -c 2 -o /tmp/reps/srcall_C1 \
  python scripts/prof_c1.py > gpurun_out/ncu_srcall_C1.log 2>&1; echo srcall_C1=$?
ncu -i /tmp/reps/srcall_C1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/reps/srcall_C1.csv 2>&1
python scripts/src_conflicts.py /tmp/reps/srcall_C1.csv 12 > gpurun_out/conflicts_C1.txt 2>&1
cat gpurun_out/conflicts_C*.txt
