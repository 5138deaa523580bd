timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ay_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2ay_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_BAR_ACQREL=1" > gpurun_out/r2ay_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2ay_variants.txt
timeout 600 python tools/levels.py C2 2 2>&1 | tail -20
