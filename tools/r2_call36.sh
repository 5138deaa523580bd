# row records everywhere (heads removed; multi-rank blocks and 64-bit-offset graphs too)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ak_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2ak_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_DENSE=1" > gpurun_out/r2ak_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2ak_variants.txt
timeout 900 python tools/team_bench.py C2 > gpurun_out/r2ak_team_C2.txt 2>&1; tail -6 gpurun_out/r2ak_team_C2.txt
