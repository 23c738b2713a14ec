# r2_prof3.sh : ncu launch lists + full captures of C2 / C3 / C4 / C1 on the current kernels, summarised ON THE BOX
mkdir -p gpurun_out /tmp/reps
for cfg in C2 C3 C4; do
  CONFIG=$cfg MAXIT=2 python scripts/prof_c2.py > gpurun_out/prof_plain_$cfg.log 2>&1 || { echo plain_failed_$cfg; continue; }
  CONFIG=$cfg MAXIT=2 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$cfg.csv python scripts/prof_c2.py > gpurun_out/ncu_ll_$cfg.log 2>&1; echo ll_$cfg=$?
  CONFIG=$cfg MAXIT=1 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_row|k_col|k_hartley|k_t_filter|k_axpy_dev" -s 5 -c 9 -o /tmp/reps/full_$cfg \
    python scripts/prof_c2.py > gpurun_out/ncu_full_$cfg.log 2>&1; echo full_$cfg=$?
done
python scripts/prof_c1.py > gpurun_out/prof_c1_plain.log 2>&1 || { echo plain_failed_c1; }
ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C1.csv \
  python scripts/prof_c1.py > gpurun_out/ncu_ll_C1.log 2>&1; echo ll_C1=$?
ncu -f --set full --import-source on --clock-control none -k regex:"k_row|k_col|k_pfa" -o /tmp/reps/full_C1 \
  python scripts/prof_c1.py > gpurun_out/ncu_full_C1.log 2>&1; echo full_C1=$?
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_new.json
python scripts/ncu_summary.py full /tmp/reps/full_C2.ncu-rep gpurun_out/r02_ncu_full_c2.csv gpurun_out/ncu_traffic_new.json "256 256 256" C2 > /dev/null
python scripts/ncu_summary.py full /tmp/reps/full_C1.ncu-rep gpurun_out/r02_ncu_full_c1.csv gpurun_out/ncu_traffic_new.json "256 1023 1023" C1 > /dev/null
python scripts/ncu_summary.py full /tmp/reps/full_C3.ncu-rep gpurun_out/r02_ncu_full_c3.csv gpurun_out/ncu_traffic_new.json "128 512 512" C3 > /dev/null
python scripts/ncu_summary.py full /tmp/reps/full_C4.ncu-rep gpurun_out/r02_ncu_full_c4.csv gpurun_out/ncu_traffic_new.json "128 1024 1024" C4 > /dev/null
for c in C1 C2 C3 C4; do python scripts/ncu_summary.py stalls /tmp/reps/full_$c.ncu-rep gpurun_out/r02_stalls_$(echo $c | tr A-Z a-z).txt $c > /dev/null; done
# source-level hot spots of the dominant kernel (C2 K2) and of C1's column matvec pass
ncu -i /tmp/reps/full_C2.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_colc > gpurun_out/src_c2_k2.csv 2>&1
for c in C2 C3 C4 C1; do ncu -i /tmp/reps/full_$c.ncu-rep --page raw --csv > gpurun_out/raw_$c.csv 2>&1; done
ls -la gpurun_out
