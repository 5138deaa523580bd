# final-state evidence (code after the multi-rank fixes): Table-2 ablation, RGG24, bench, ncu
timeout 1200 python tools/ablation.py K21 > gpurun_out/r2ap_ablation_K21.md 2>&1; tail -12 gpurun_out/r2ap_ablation_K21.md
timeout 1200 python tools/ablation.py C2 > gpurun_out/r2ap_ablation_C2.md 2>&1; tail -12 gpurun_out/r2ap_ablation_C2.md
timeout 1200 python tools/big_check.py RGG24 4 > gpurun_out/r2ap_big_RGG24.txt 2>&1; tail -4 gpurun_out/r2ap_big_RGG24.txt
TAG=r2h bash tools/evidence_r1c.sh
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo smoke=$?
