#!/bin/bash
# One GPU iteration: parity tests, per-level timings, bench.  Usage: tools/gpu_iter.sh TAG [pytest -k expr]
TAG=${1:-iter}; K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -x -q --tb=short -k "$K" > gpurun_out/tests_$TAG.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/tests_$TAG.log 2>&1; fi
echo "tests_rc=$?"; tail -15 gpurun_out/tests_$TAG.log
timeout 300 python tools/levels.py C2 4 > gpurun_out/levels_c2_$TAG.txt 2>&1; cat gpurun_out/levels_c2_$TAG.txt
timeout 300 python tools/levels.py C4 1 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
