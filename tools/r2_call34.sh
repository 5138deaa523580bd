REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_DENSE_TAIL=0" "PP_DENSE_TAIL=16" "PP_DENSE_TAIL=32" "PP_DENSE_TAIL=64" > gpurun_out/r2ai_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L" gpurun_out/r2ai_variants.txt
