# persistent SSSP (one cooperative launch): parity, timing, smoke; bench with the record design model
timeout 900 python -m pytest tests/test_gpu_sssp.py -x -q > gpurun_out/r2g_tests_sssp.log 2>&1; echo sssp_tests=$?; tail -2 gpurun_out/r2g_tests_sssp.log
timeout 600 python tools/sssp_bench.py C2 4 > gpurun_out/r2g_sssp_bench_C2.txt 2>&1; tail -4 gpurun_out/r2g_sssp_bench_C2.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo smoke=$?; cat gpurun_out/r2g_smoke.log | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_sssp_launches.csv python tools/sssp_bench.py C2 1 > /dev/null 2>&1; echo ncu=$?
timeout 600 python bench.py > gpurun_out/r2g_bench_C2.json 2> gpurun_out/r2g_bench.err; cat gpurun_out/r2g_bench_C2.json
