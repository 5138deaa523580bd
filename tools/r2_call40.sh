timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ao_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2ao_tests.log
timeout 900 python tools/team_bench.py C2 > gpurun_out/r2ao_team_C2.txt 2>&1; grep -E "engine|team" gpurun_out/r2ao_team_C2.txt
timeout 900 python tools/team_bench.py C5 1,2,4,8 4 > gpurun_out/r2ao_team_C5.txt 2>&1; grep -E "engine|team" gpurun_out/r2ao_team_C5.txt
