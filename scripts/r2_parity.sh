grep -E "MemTotal|MemAvailable" /proc/meminfo > gpurun_out/meminfo.txt

timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -s --durations=0 > gpurun_out/fullsize.log 2>&1; echo full_rc=$?; tail -25 gpurun_out/fullsize.log
