REPS=1 STEPS=64 C4=1 tools/variants.sh "PP_BFS_BLOCK=1024" "PP_BFS_BLOCK=768" "PP_BFS_BLOCK=512" > gpurun_out/r2bd_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L" gpurun_out/r2bd_variants.txt
