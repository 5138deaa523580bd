REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_BAR_SLEEP=16" "PP_BAR_SLEEP=0" "PP_BAR_SLEEP=64" "PP_LOWLAT_EDGES=131072" "PP_LOWLAT_EDGES=8192" > gpurun_out/r2bb_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2bb_variants.txt
