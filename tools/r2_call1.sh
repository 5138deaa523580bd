set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/micro/gridbar 4000 > gpurun_out/gridbar.txt 2>&1; cat gpurun_out/gridbar.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.log 2>&1; tail -3 gpurun_out/r2a_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2a_bench.json 2>gpurun_out/r2a_bench.err; cat gpurun_out/r2a_bench.json | head -c 600
