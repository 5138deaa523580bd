# dense pull: shared-memory footprint (L1 carve-out) sweep
REPS=1 STEPS=64 C4=1 tools/variants.sh "PP_DENSE=0 PP_RQ_EXTRA=64" "PP_DENSE=0 PP_RQ_EXTRA=32" "PP_DENSE=1 PP_DENSE_R=3 PP_DENSE_U=1" "PP_DENSE=1 PP_DENSE_R=2 PP_DENSE_U=1" "PP_DENSE=1 PP_DENSE_R=4 PP_DENSE_U=1" "PP_DENSE=1 PP_DENSE_R=3 PP_DENSE_U=1 PP_DENSE_MIN8=5" "PP_DENSE=1 PP_DENSE_R=3 PP_DENSE_U=1 PP_CHUNK=64 PP_HEAVY=64" "PP_DENSE=0 PP_CHUNK=64 PP_HEAVY=64" > gpurun_out/r2u_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L|Error|error" gpurun_out/r2u_variants.txt
