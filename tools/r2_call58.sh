# final HEAD (768-thread CTAs): ncu full + launch list, bench (+reference), levels
TAG=r2j
CAP="ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --model-sources 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 3 -c 1 -f -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --model-sources 0 > gpurun_out/${TAG}_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep gpurun_out/ncu_C2.json "$CAP" "$TAG" && cp gpurun_out/ncu_C2.json profiles/ncu_C2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --model-sources 0 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C2.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench_C2.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2> /dev/null
timeout 300 python tools/levels.py C2 8 > gpurun_out/${TAG}_levels_C2.txt 2>&1
timeout 300 python tools/levels.py C4 1 > gpurun_out/${TAG}_levels_C4.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$?
