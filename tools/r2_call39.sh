# multi-rank: warp-aggregated list slots; dense pull on blocks on / off
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_dist_mp.py -x -q 2>&1 | tail -1
for v in "PP_DENSE_DIST=1" "PP_DENSE_DIST=0"; do
  echo "=== $v"; env $v python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
  timeout 900 python tools/team_bench.py C2 1,2,8 > gpurun_out/r2an_team_C2_$v.txt 2>&1; grep team gpurun_out/r2an_team_C2_$v.txt
  timeout 900 python tools/team_bench.py C5 1,2,8 4 > gpurun_out/r2an_team_C5_$v.txt 2>&1; grep team gpurun_out/r2an_team_C5_$v.txt
done
