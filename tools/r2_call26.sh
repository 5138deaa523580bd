# cleaned defaults (dense ring R1, sparse pull on records, 64-edge chunks): full GPU suite, bench,
# per-level table, ncu of the heaviest push and of the dense heavy pull
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2aa_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2aa_tests.log
timeout 600 python bench.py > gpurun_out/r2aa_bench.json 2> gpurun_out/r2aa_bench.err; cat gpurun_out/r2aa_bench.json
timeout 600 python tools/levels.py C2 8 > gpurun_out/r2aa_levels_c2.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bfs_persistent --launch-skip 4 --launch-count 1 -o gpurun_out/r2aa_push python tools/prof_level.py C2 push 5 > gpurun_out/r2aa_push.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bfs_persistent --launch-skip 4 --launch-count 1 -o gpurun_out/r2aa_pull python tools/prof_level.py C2 pull 5 > gpurun_out/r2aa_pull.log 2>&1; echo ncu2=$?
