timeout 900 python -m pytest tests/test_gpu_sssp.py -x -q 2>&1 | tail -1
timeout 600 python tools/sssp_bench.py C2 4 > gpurun_out/r2h_sssp_bench_C2.txt 2>&1; grep summary gpurun_out/r2h_sssp_bench_C2.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_sssp_launches.csv python tools/sssp_bench.py C2 1 0.01 > /dev/null 2>&1; echo ncu=$?
