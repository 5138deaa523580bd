for v in "PP_STREAM_U=4" "PP_STREAM_U=8" "PP_STREAM_U=16"; do
  echo "=== $v"
  env $v python paper_1804_03327_b200/build.py 1 >/dev/null 2>&1 || { echo build failed; continue; }
  timeout 600 python tools/c3_sweep.py --reps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['arm']!='masked_ee' and d['rho'] in (0.01,0.1,1.0): print(d['u'],d['arm'],d['rho'],round(d['us'],1),round(d['frac'],3))"
done
