# dense pull: ring (R1) vs register prefetch; L1 carve-out control (pad = the ring's 33 KB)
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_DENSE_R=1" "PP_DENSE_REG=1" "PP_DENSE=0" "PP_DENSE=0 PP_SMEM_PAD=33792" "PP_DENSE_REG=1 PP_DENSE_RB=1" > gpurun_out/r2y_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L|Error|error" gpurun_out/r2y_variants.txt
