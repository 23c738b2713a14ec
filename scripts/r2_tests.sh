timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/tests_all.log 2>&1; echo tests_rc=$?
tail -25 gpurun_out/tests_all.log
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
