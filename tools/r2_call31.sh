# round-2 final-state evidence (dense pull): tests, ncu full + launch list, bench (+reference),
# levels, smoke, paper-graph analogs
TAG=r2f bash tools/evidence_r1c.sh
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke_rc=$?
for c in C2_ef64 S23E32 S24E16 K21; do timeout 900 python tools/big_check.py $c 16 > gpurun_out/r2f_big_$c.txt 2>&1; done
timeout 1200 python tools/big_check.py C5 4 > gpurun_out/r2f_big_C5.txt 2>&1
tail -3 gpurun_out/r2f_big_*.txt
