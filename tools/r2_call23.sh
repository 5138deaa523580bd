# dense pull: words per step (U) x ring depth (R), item size 16
REPS=1 STEPS=64 C4=1 tools/variants.sh "PP_DENSE_U=1" "PP_DENSE_U=2 PP_DENSE_R=2" "PP_DENSE_U=2 PP_DENSE_R=3" "PP_DENSE_U=2 PP_DENSE_R=4" "PP_DENSE_IW=16" "PP_DENSE_U=1 PP_DENSE_R=2" > gpurun_out/r2x_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L|Error|error" gpurun_out/r2x_variants.txt
