# r2_exp3.sh : PFA solve after the DFT_31 / mirror-slot / scratch changes, lanes-per-CTA variants
mkdir -p gpurun_out
for v in base g3 g3c7 base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1907_13428_b200/lib/libfdg.so; else lib=$PWD/paper_1907_13428_b200/lib/libfdg_$v.so; fi
  par=$(FDG_LIB=$lib timeout 300 python -m pytest tests/test_gpu_c1.py -q -m gpu -x -k "precond or full_size" 2>&1 | tail -1)
  b=$(FDG_LIB=$lib timeout 300 python scripts/bench_c1.py 2>&1 | tail -1)
  echo "$v | $par | $b"
done 2>&1 | tee gpurun_out/exp3_pfa.txt
