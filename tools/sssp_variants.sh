#!/bin/bash
# SSSP light-row group size sweep on one B200: rebuild with PP_SSSP_G and time C2.
mkdir -p gpurun_out
for G in 4 16 8; do
  PP_SSSP_G=$G python paper_1804_03327_b200/build.py > /dev/null 2>&1 || { echo "build G=$G failed"; continue; }
  echo "G=$G"; timeout 300 python tools/sssp_bench.py C2 4 0.01 | grep summary
done
