REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_CTR_SPREAD=0" "PP_CTR_SPREAD=1" > gpurun_out/r2az_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2az_variants.txt
