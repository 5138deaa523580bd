timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2l_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2l_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value'],1), round(d['roofline']['frac'],4))"
