python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/quick_check.py 2>&1 | tail -1
timeout 300 python tools/cta_balance.py C2 2 > gpurun_out/r2i_cta_C2.txt 2>&1; cat gpurun_out/r2i_cta_C2.txt
timeout 300 python tools/cta_balance.py C4 1 > gpurun_out/r2i_cta_C4.txt 2>&1; head -14 gpurun_out/r2i_cta_C4.txt
timeout 300 python tools/levels.py C4 1 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 64 --model-sources 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value'],1), 'GTEPS', round(d['ms_per_step']*1e3,1), 'us', d['clocks'])"
