# dense pull: item size, speculative probes, row-begin record (defaults now R1 U1, chunk 64)
REPS=1 STEPS=64 C4=1 tools/variants.sh "PP_DENSE_IW=8" "PP_DENSE_IW=2" "PP_DENSE_IW=1" "PP_DENSE_SPEC=1" "PP_DENSE_RB=1" "PP_DENSE_IW=2 PP_DENSE_SPEC=1 PP_DENSE_RB=1" > gpurun_out/r2w_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L|Error|error" gpurun_out/r2w_variants.txt
