python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_dist_mp.py -x -q --tb=short > gpurun_out/r2l_mp.log 2>&1; tail -15 gpurun_out/r2l_mp.log
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short --deselect tests/test_gpu_dist_mp.py::test_two_processes_ipc_bit_exact > gpurun_out/r2l_tests.log 2>&1; tail -5 gpurun_out/r2l_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; tail -2 gpurun_out/r2l_smoke.log
