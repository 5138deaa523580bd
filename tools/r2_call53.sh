# round-2 final evidence at HEAD
TAG=r2i bash tools/evidence_r1c.sh
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo smoke=$?
for c in C2_ef64 S23E32 S24E16 K21; do timeout 900 python tools/big_check.py $c 16 > gpurun_out/r2i_big_$c.txt 2>&1; done
timeout 1200 python tools/big_check.py C5 4 > gpurun_out/r2i_big_C5.txt 2>&1
timeout 1200 python tools/big_check.py RGG24 4 > gpurun_out/r2i_big_RGG24.txt 2>&1
timeout 900 python tools/team_bench.py C5 1,2,4,8 4 > gpurun_out/r2i_team_C5.txt 2>&1
timeout 600 python tools/sssp_bench.py C2 4 > gpurun_out/r2i_sssp_bench_C2.txt 2>&1
timeout 1200 python tools/ablation.py K21 C2 > gpurun_out/r2i_ablation.md 2>&1
echo done
