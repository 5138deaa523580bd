REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_ONE_PUSH=0 PP_ONE_RESID=0" "PP_ONE_PUSH=1 PP_ONE_RESID=0" "PP_ONE_PUSH=0 PP_ONE_RESID=1" "PP_ONE_PUSH=1 PP_ONE_RESID=1" > gpurun_out/r2ae_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L" gpurun_out/r2ae_variants.txt
