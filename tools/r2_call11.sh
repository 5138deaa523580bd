C4=1 REPS=2 STEPS=64 tools/variants.sh "PP_PUSH_KU=4" "PP_PUSH_KU=2" > gpurun_out/r2k_variants.txt 2>&1
grep -E "variant|BENCH|per-level|quick" gpurun_out/r2k_variants.txt
python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
echo "== narrow start on C2"; PP_NARROW=1 timeout 300 python tools/levels.py C2 2 2>&1 | head -24
PP_NARROW=1 timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 64 --model-sources 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH narrow', round(d['value'],1), 'GTEPS', round(d['ms_per_step']*1e3,1), 'us')"
echo "== C3 unmasked stream: plain vs relabelled"
timeout 600 python tools/c3_sweep.py --unmasked-only --reps 10 2>&1 | head -2
timeout 600 python tools/c3_sweep.py --unmasked-only --reps 10 --relabel 2>&1 | head -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mxv_pull_stream --launch-skip 2 --launch-count 1 -f -o gpurun_out/r2k_stream python tools/c3_sweep.py --unmasked-only --reps 3 > gpurun_out/r2k_stream.log 2>&1; tail -2 gpurun_out/r2k_stream.log
