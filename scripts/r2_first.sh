nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ldconfig -p | grep -i fftw > gpurun_out/fftw_host.txt; echo fftw_rc=$? >> gpurun_out/fftw_host.txt
lscpu > gpurun_out/lscpu.txt
bash scripts/quick.sh
timeout 300 python scripts/iter_slope.py > gpurun_out/slope_c2.txt 2>&1
timeout 300 python scripts/iter_slope.py 128 512 512 > gpurun_out/slope_c3.txt 2>&1
tail -2 gpurun_out/slope_c2.txt gpurun_out/slope_c3.txt
