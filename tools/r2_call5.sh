REPS=2 tools/variants.sh "PP_STEAL=0" "PP_PULL_PF=1" "PP_STEAL=4" "PP_STEAL=4 PP_PULL_PF=1" "PP_STEAL=16" > gpurun_out/r2e_variants.txt 2>&1
cat gpurun_out/r2e_variants.txt
