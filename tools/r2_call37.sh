timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2al_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2al_tests.log
timeout 900 python tools/team_bench.py C2 > gpurun_out/r2al_team_C2.txt 2>&1; tail -8 gpurun_out/r2al_team_C2.txt
