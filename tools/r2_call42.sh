# init overlap: parity, then A/B
timeout 1500 python -m pytest tests/test_gpu_bfs.py tests/test_gpu_fullsize.py tests/test_gpu_mxv.py -q -x > gpurun_out/r2aq_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2aq_tests.log
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_INIT_OVERLAP=0" "PP_INIT_OVERLAP=1" > gpurun_out/r2aq_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|init" gpurun_out/r2aq_variants.txt | head -40
timeout 300 python tools/levels.py C2 2 2>&1 | head -20
