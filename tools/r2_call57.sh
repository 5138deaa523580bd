timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2be_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2be_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_BFS_BLOCK=768" "PP_BFS_BLOCK=1024" > gpurun_out/r2be_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level" gpurun_out/r2be_variants.txt
python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 900 python tools/big_check.py RGG24 4 2>&1 | tail -4
timeout 900 python bench.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['roofline']['frac'], d['step_ms'])"
