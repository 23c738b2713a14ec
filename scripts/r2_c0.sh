for pdl in 0 1; do echo "graph nmax default, FDG_PDL_MASK=$pdl"; FDG_PDL_MASK=$([ $pdl = 1 ] && echo 62 || echo 0) python scripts/c0_probe.py 3; done
FDG_PCG_GRAPH_NMAX=0 python scripts/c0_probe.py 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c0_launches.csv python scripts/c0_probe.py 1 > gpurun_out/c0_ncu.log 2>&1; echo ncu_rc=$?
