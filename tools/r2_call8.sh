C4=1 REPS=2 STEPS=64 tools/variants.sh "PP_LOWLAT_VREC=0 PP_PF_ROWS=0" "PP_PF_ROWS=0" "PP_LOWLAT_VREC=0" "PP_LOWLAT_VREC=1" > gpurun_out/r2h_variants.txt 2>&1
grep -E "variant|BENCH|per-level|quick" gpurun_out/r2h_variants.txt
