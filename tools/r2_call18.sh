REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_PUSH_KU=2" "PP_PUSH_KU=1" "PP_PULL_KC=2" "PP_BFS_BLOCK=768" "PP_LOWLAT_VREC=1" "PP_PULL_PF=1" > gpurun_out/r2r_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|Error" gpurun_out/r2r_variants.txt
