# r2_prof1.sh : ncu evidence for C1 (PFA solve + matvec), C3 and C4 (one PCG iteration's kernels)
mkdir -p gpurun_out
bash scripts/ncu_c1.sh
bash scripts/ncu_cfg.sh C3
bash scripts/ncu_cfg.sh C4
ls -la gpurun_out/
