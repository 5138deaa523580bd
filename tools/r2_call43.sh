REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_LOWLAT_VREC=0" "PP_LOWLAT_VREC=1" > gpurun_out/r2ar_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2ar_variants.txt
tools/variants_levels.sh "PP_LOWLAT_VREC=0" "PP_LOWLAT_VREC=1" > gpurun_out/r2ar_levels.txt 2>&1; cat gpurun_out/r2ar_levels.txt
