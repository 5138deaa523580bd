C4=1 REPS=2 STEPS=64 tools/variants.sh "PP_FUSED_SYNC=0" "PP_FUSED_SYNC=1" > gpurun_out/r2g_variants.txt 2>&1
grep -E "variant|BENCH|per-level|quick" gpurun_out/r2g_variants.txt
python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 300 python tools/cta_balance.py C2 2 > gpurun_out/r2g_cta_C2.txt 2>&1; head -20 gpurun_out/r2g_cta_C2.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent --launch-skip 3 --launch-count 1 -f -o gpurun_out/r2g_c4 python tools/levels.py C4 1 > gpurun_out/r2g_c4.log 2>&1; tail -2 gpurun_out/r2g_c4.log
