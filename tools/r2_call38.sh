# dense pull on multi-rank blocks: team / two-process parity, full suite, team bench
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2am_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2am_tests.log
timeout 900 python tools/team_bench.py C2 > gpurun_out/r2am_team_C2.txt 2>&1; tail -6 gpurun_out/r2am_team_C2.txt
timeout 900 python tools/team_bench.py C5 1,2,4,8 4 > gpurun_out/r2am_team_C5.txt 2>&1; tail -6 gpurun_out/r2am_team_C5.txt
