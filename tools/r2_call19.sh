# dense pull (bulk-copy rings): parity first, then A/B variants
timeout 300 python tools/quick_check.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_bfs.py -x -q 2>&1 | tail -3
REPS=1 STEPS=64 C4=1 tools/variants.sh "PP_DENSE=0" "PP_DENSE=1" "PP_DENSE=1 PP_DENSE_U=1" "PP_DENSE=1 PP_DENSE_R=3 PP_DENSE_U=1" "PP_DENSE=1 PP_DENSE_MIN8=1" "PP_DENSE=1 PP_DENSE_MIN8=4" > gpurun_out/r2t_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L|Error|error" gpurun_out/r2t_variants.txt
