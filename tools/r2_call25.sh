# sparse pull reading the dense records (L2 reuse after a dense level); parity of that build
PP_SPARSE_REC=1 python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_bfs.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
REPS=2 STEPS=64 C4=1 tools/variants.sh "PP_SPARSE_REC=0" "PP_SPARSE_REC=1" > gpurun_out/r2z_variants.txt 2>&1
grep -E "variant|BENCH|quick|per-level|L3 L|L4 L|Error|error" gpurun_out/r2z_variants.txt
