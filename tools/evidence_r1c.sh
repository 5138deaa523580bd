#!/bin/bash
# Round-1 (second half) evidence on one B200: GPU tests, ncu full capture + launch list, bench, levels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG:-r1c}_tests_gpu.log 2>&1; tail -2 gpurun_out/${TAG:-r1c}_tests_gpu.log
CAP="ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --model-sources 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 3 -c 1 -f -o gpurun_out/${TAG:-r1c}_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --model-sources 0 > gpurun_out/${TAG:-r1c}_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG:-r1c}_full.ncu-rep gpurun_out/ncu_C2.json "$CAP" "${TAG:-r1c}" && cp gpurun_out/ncu_C2.json profiles/ncu_C2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-r1c}_launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --model-sources 0 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${TAG:-r1c}_bench_C2.json 2> gpurun_out/${TAG:-r1c}_bench.err; cat gpurun_out/${TAG:-r1c}_bench_C2.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG:-r1c}_bench_reference.json 2> gpurun_out/${TAG:-r1c}_bench_reference.err
timeout 300 python tools/levels.py C2 8 > gpurun_out/${TAG:-r1c}_levels_C2.txt 2>&1
timeout 300 python tools/levels.py C4 1 > gpurun_out/${TAG:-r1c}_levels_C4.txt 2>&1
