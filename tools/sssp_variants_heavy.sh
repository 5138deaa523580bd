#!/bin/bash
# SSSP heavy-row threshold sweep on one B200: rebuild with PP_SSSP_HEAVY, time C2.
for H in 64 128 512 256; do
  PP_SSSP_HEAVY=$H python paper_1804_03327_b200/build.py > /dev/null 2>&1 || { echo "build H=$H failed"; continue; }
  echo "H=$H"; timeout 300 python tools/sssp_bench.py C2 4 0.01 | grep summary
done
