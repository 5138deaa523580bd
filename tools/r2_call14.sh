REPS=2 STEPS=64 tools/variants.sh "PP_PULL_REC=0" "PP_PULL_REC=1" "PP_PULL_REC=1 PP_PULL_KC=2" > gpurun_out/r2n_variants.txt 2>&1
grep -E "variant|BENCH|quick|L3 L|L4 L.*c=  1705702" gpurun_out/r2n_variants.txt
