# ncu_cfg.sh CONFIG : launch list of a 2-iteration PCG solve and a full capture of one iteration's
# kernels (K1F K2 K3 P1-P5 + the x update) of a BASELINE config -> gpurun_out/ncu_CONFIG.*
# (the plain command runs first and must exit 0; never a bench number under ncu)
cfg=${1:-C2}
CONFIG=$cfg MAXIT=2 python scripts/prof_c2.py > gpurun_out/prof_plain_$cfg.log 2>&1 || { echo plain_failed; exit 1; }
CONFIG=$cfg MAXIT=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$cfg.csv python scripts/prof_c2.py > gpurun_out/ncu_ll_$cfg.log 2>&1
echo ll_rc=$?
CONFIG=$cfg MAXIT=1 ncu --set full --import-source on --clock-control none \
  -k regex:"k_row|k_col|k_hartley|k_t_filter|k_axpy_dev" -s 5 -c 9 -o gpurun_out/full_$cfg \
  python scripts/prof_c2.py > gpurun_out/ncu_full_$cfg.log 2>&1
echo full_rc=$?
