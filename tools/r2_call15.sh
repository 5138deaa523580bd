C4=1 REPS=2 STEPS=64 tools/variants.sh "PP_FAST_NTH=0" "PP_FAST_NTH=1" > gpurun_out/r2o_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L.*c=  1705702" gpurun_out/r2o_variants.txt
python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 600 python tools/c3_sweep.py --unmasked-only --reps 10 2>&1 | head -1
