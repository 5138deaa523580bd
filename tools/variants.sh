#!/bin/bash
# Build and time compile-time variants (GPU box), each checked for parity first.
# Usage: tools/variants.sh "ENV1" "ENV2" ...   (REPS=2 runs the whole list twice, alternating)
for rep in $(seq 1 ${REPS:-1}); do
for v in "$@"; do
  echo "=== variant: $v (pass $rep)"
  env $v python paper_1804_03327_b200/build.py 1 >/dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python tools/quick_check.py 2>&1 | tail -1
  timeout 300 python tools/levels.py C2 4 2>&1 | grep -E "^src|L3 L|L4 L"
  if [ -n "$C4" ]; then timeout 300 python tools/levels.py C4 1 2>&1 | grep -E "^src|per-level" | head -4; fi
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps ${STEPS:-64} --model-sources 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value'],1), 'GTEPS', round(d['ms_per_step']*1e3,1), 'us')"
done
done
