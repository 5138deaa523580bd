REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_PUSH_KU=2" "PP_PUSH_KU=4 PP_CHUNK=128 PP_HEAVY=64" > gpurun_out/r2bg_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2bg_variants.txt
