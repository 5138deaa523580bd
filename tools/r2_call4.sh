set -x

timeout 300 python -m pytest tests/test_gpu_bfs.py -x -q --tb=short -k debug_level > gpurun_out/r2d_debuglevel.log 2>&1; tail -3 gpurun_out/r2d_debuglevel.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent --launch-skip 4 --launch-count 1 -f -o gpurun_out/r2d_pull python tools/prof_level.py C2 pull 5 > gpurun_out/r2d_pull.log 2>&1; tail -3 gpurun_out/r2d_pull.log
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:bfs_persistent --launch-skip 4 --launch-count 1 -f -o gpurun_out/r2d_pull_nocc python tools/prof_level.py C2 pull 5 > gpurun_out/r2d_pull_nocc.log 2>&1; tail -3 gpurun_out/r2d_pull_nocc.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent --launch-skip 4 --launch-count 1 -f -o gpurun_out/r2d_push python tools/prof_level.py C2 push 5 > gpurun_out/r2d_push.log 2>&1; tail -3 gpurun_out/r2d_push.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bfs_persistent --csv --log-file gpurun_out/r2d_levels_alone.csv python tools/prof_level.py C2 pull 5 > /dev/null 2>&1; echo done
