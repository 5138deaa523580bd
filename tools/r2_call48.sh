timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2aw_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2aw_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
