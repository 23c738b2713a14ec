# plain run first (must exit 0), then the per-launch device-time list of one short bench
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --admm-steps 0 --profile-reps 1 --configs "" > gpurun_out/ll_plain.json 2> gpurun_out/ll_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --admm-steps 0 --profile-reps 1 --configs "" > gpurun_out/ll_ncu.log 2>&1
echo rc=$?
