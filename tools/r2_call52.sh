timeout 900 python -m pytest tests/test_gpu_sssp.py -q -x 2>&1 | tail -1
timeout 600 python tools/sssp_bench.py C2 4 0.01 2>&1 | grep summary
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_BAR_PRESYNC=0" "PP_BAR_PRESYNC=1" > gpurun_out/r2ba_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2ba_variants.txt
