timeout 300 python tools/quick_check.py 2>&1 | tail -1
timeout 600 python tools/cta_balance.py C2 2 2>&1 | head -20
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_DENSE=1" > gpurun_out/r2av_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2av_variants.txt
timeout 300 python tools/levels.py C2 2 2>&1 | tail -3
