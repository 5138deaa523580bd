REPS=2 STEPS=64 tools/variants.sh "PP_DENSE_MIN8=2" "PP_DENSE_MIN8=1" "PP_DENSE_MIN8=3" "PP_DENSE_IW=4" > gpurun_out/r2bc_variants.txt 2>&1
grep -E "variant|BENCH|quick|L3 L|L4 L" gpurun_out/r2bc_variants.txt
python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:bfs_persistent -s 3 -c 1 -o gpurun_out/r2bc_full_cachenone python bench.py --steps 1 --warmup 3 --no-cpu-baseline --model-sources 0 > gpurun_out/r2bc_ncu.log 2>&1; echo ncu=$?
