#!/bin/bash
# Per-level tables of 2 C2 sources and the C4 per-level mean for each compile-time variant.
for v in "$@"; do
  echo "=== variant: $v"
  env $v python paper_1804_03327_b200/build.py 1 >/dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python tools/quick_check.py 2>&1 | tail -1
  timeout 300 python tools/levels.py C2 2 2>&1 | grep -E "^src|^   L|isolated"
  timeout 300 python tools/levels.py C4 1 2>&1 | grep -E "per-level|isolated"
done
