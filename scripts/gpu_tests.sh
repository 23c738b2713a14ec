timeout 900 python -m pytest tests -q -m gpu -x -s > gpurun_out/tests_all.log 2>&1; echo tests_rc=$?
grep -E "gpu steps|passed|failed|FAILED" gpurun_out/tests_all.log | tail -5
