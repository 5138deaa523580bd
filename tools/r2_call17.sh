REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_PUSH_KU=2" "PP_PUSH_KU=2 PP_FUSED_SYNC=0" "PP_PUSH_KU=2 PP_SUM_WORDS=4096 PP_SUM_RESID=1" "PP_PUSH_KU=2 PP_SUM_WORDS=2048 PP_SUM_RESID=1" "PP_PUSH_KU=4" > gpurun_out/r2q_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|Error" gpurun_out/r2q_variants.txt
