python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_mxv.py -x -q --tb=short > gpurun_out/r2m_mxv.log 2>&1; tail -3 gpurun_out/r2m_mxv.log
timeout 900 python tools/c3_sweep.py --reps 10 --out gpurun_out/r2m_c3.jsonl > /dev/null 2>&1; python -c "
import json
for l in open('gpurun_out/r2m_c3.jsonl'):
    d=json.loads(l)
    if d['arm']!='masked_ee' and d['rho'] in (0.01,0.1,1.0): print(d['u'],d['arm'],d['rho'],round(d['us'],1),round(d['frac'],3))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mxv_pull_stream --launch-skip 2 --launch-count 1 -f -o gpurun_out/r2m_stream python tools/c3_sweep.py --unmasked-only --reps 3 > gpurun_out/r2m_stream.log 2>&1; tail -1 gpurun_out/r2m_stream.log
timeout 600 python tools/fig2_sweep.py K21 5 2>&1 | head -13
