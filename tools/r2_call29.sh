# code-size cut (ablation kernel split, one push_round / residual call site): parity + timing
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ad_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2ad_tests.log
tools/variants_levels.sh "PP_DENSE=1" > gpurun_out/r2ad_levels.txt 2>&1; cat gpurun_out/r2ad_levels.txt
REPS=2 STEPS=64 tools/variants.sh "PP_DENSE=1" > gpurun_out/r2ad_variants.txt 2>&1
grep -E "variant|BENCH|quick" gpurun_out/r2ad_variants.txt
