tools/variants_levels.sh "PP_DENSE=1" "PP_DENSE=0" "PP_CHUNK=128 PP_HEAVY=128" "PP_NOINLINE_PULL=1" "PP_DENSE=0 PP_CHUNK=128 PP_HEAVY=128" > gpurun_out/r2ab_levels.txt 2>&1
cat gpurun_out/r2ab_levels.txt
