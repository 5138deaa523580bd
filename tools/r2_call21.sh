# dense pull: ring depth 1/2, never-dense control (smem/code cost), chunk 64; then ncu of the dense heavy pull
REPS=1 STEPS=64 C4=1 tools/variants.sh "PP_DENSE=0 PP_CHUNK=64 PP_HEAVY=64" "PP_DENSE=1 PP_DENSE_R=1 PP_DENSE_U=1 PP_CHUNK=64 PP_HEAVY=64" "PP_DENSE=1 PP_DENSE_R=2 PP_DENSE_U=1 PP_CHUNK=64 PP_HEAVY=64" "PP_DENSE=1 PP_DENSE_R=2 PP_DENSE_U=1 PP_CHUNK=64 PP_HEAVY=64 PP_DENSE_MIN8=9" "PP_DENSE=1 PP_DENSE_R=2 PP_DENSE_U=2 PP_CHUNK=64 PP_HEAVY=64" > gpurun_out/r2v_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L|Error|error" gpurun_out/r2v_variants.txt
PP_DENSE=1 PP_DENSE_R=2 PP_DENSE_U=1 PP_CHUNK=64 PP_HEAVY=64 python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bfs_persistent --launch-skip 4 --launch-count 1 -o gpurun_out/r2v_dense_pull python tools/prof_level.py C2 pull 5 > gpurun_out/r2v_dense_pull.log 2>&1; echo ncu_rc=$?
