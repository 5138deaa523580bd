#!/bin/bash
# Round evidence on one B200: parity tests, bench (+reference arm), C3 sweep, level traces,
# ncu launch list and one full ncu capture of the BFS kernel.  Outputs gpurun_out/${TAG}_*.
TAG=${1:-r1}
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then timeout 1500 python -m pytest tests -m gpu -q --tb=short > gpurun_out/${TAG}_tests.log 2>&1; echo "tests_rc=$?"; tail -2 gpurun_out/${TAG}_tests.log; fi
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>&1; cat gpurun_out/${TAG}_bench_ref.json
timeout 600 python tools/c3_sweep.py --out gpurun_out/${TAG}_c3.jsonl > /dev/null 2>&1; echo "c3_rc=$?"; head -3 gpurun_out/${TAG}_c3.jsonl
timeout 600 python tools/levels.py C2 8 > gpurun_out/${TAG}_levels_c2.txt 2>&1
timeout 600 python tools/levels.py C4 2 > gpurun_out/${TAG}_levels_c4.txt 2>&1; tail -3 gpurun_out/${TAG}_levels_c4.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --model-sources 0 > /dev/null 2>&1; echo "ncu_list_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 3 -c 1 -o gpurun_out/${TAG}_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --model-sources 0 > gpurun_out/${TAG}_prof.log 2>&1; echo "ncu_full_rc=$?"
