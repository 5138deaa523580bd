REPS=1 STEPS=64 C4=1 tools/variants.sh "PP_FUSED_SYNC=1" "PP_FUSED_SYNC=0" "PP_FAST_NTH=0" "PP_STEAL=4" "PP_PULL_PF=1" "PP_PULL_REC=1" "PP_PULL_REC=1 PP_PULL_KC=2" "PP_LOWLAT_VREC=1" "PP_PF_ROWS=1" "PP_PUSH_KU=2" "PP_KO_DEPTH=1" "PP_KO_RESID=1" "PP_KO_PROBE=1" > gpurun_out/r2p_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L.*c=  1705702" gpurun_out/r2p_variants.txt
