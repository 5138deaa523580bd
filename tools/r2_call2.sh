set -x
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q --tb=short > gpurun_out/r2b_dist.log 2>&1; tail -30 gpurun_out/r2b_dist.log
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short --deselect tests/test_gpu_dist.py > gpurun_out/r2b_tests.log 2>&1; tail -5 gpurun_out/r2b_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench.json 2>gpurun_out/r2b_bench.err; head -c 400 gpurun_out/r2b_bench.json
