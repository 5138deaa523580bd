REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_BAR_ACQREL=0" "PP_BAR_ACQREL=1" > gpurun_out/r2ax_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2ax_variants.txt
PP_BAR_ACQREL=1 python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_bfs.py tests/test_gpu_dist.py -q -x 2>&1 | tail -1
timeout 300 python tools/levels.py C2 1 2>&1 | tail -2
