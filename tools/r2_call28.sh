tools/variants_levels.sh "PP_DENSE_RB=0" "PP_DENSE_RB=1" > gpurun_out/r2ac_levels.txt 2>&1
cat gpurun_out/r2ac_levels.txt
REPS=2 STEPS=64 tools/variants.sh "PP_DENSE_RB=0" "PP_DENSE_RB=1" > gpurun_out/r2ac_variants.txt 2>&1
grep -E "variant|BENCH|quick" gpurun_out/r2ac_variants.txt
