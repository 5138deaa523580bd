REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_BFS_BLOCK=768" "PP_BFS_BLOCK=640" "PP_BFS_BLOCK=896" > gpurun_out/r2bf_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2bf_variants.txt
