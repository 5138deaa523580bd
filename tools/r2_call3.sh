set -x
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2>gpurun_out/r2c_bench.err; cat gpurun_out/r2c_bench.json; tail -3 gpurun_out/r2c_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2c_bench_ref.json 2>&1; cat gpurun_out/r2c_bench_ref.json
timeout 900 python tools/team_bench.py C2 1,2,4,8 8 > gpurun_out/r2c_team_C2.txt 2>&1; cat gpurun_out/r2c_team_C2.txt
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q --tb=short > gpurun_out/r2c_fullsize.log 2>&1; tail -5 gpurun_out/r2c_fullsize.log
timeout 1500 python tools/team_bench.py C5 1,2,4,8 4 > gpurun_out/r2c_team_C5.txt 2>&1; cat gpurun_out/r2c_team_C5.txt
