for c in C2_ef64 S23E32 S24E16 K21; do timeout 900 python tools/big_check.py $c 16 > gpurun_out/r2k_big_$c.txt 2>&1; done
timeout 1200 python tools/big_check.py C5 4 > gpurun_out/r2k_big_C5.txt 2>&1
timeout 1200 python tools/big_check.py RGG24 4 > gpurun_out/r2k_big_RGG24.txt 2>&1
python tools/paper_graphs_table.py gpurun_out/r2k_big_C2_ef64.txt gpurun_out/r2k_big_S23E32.txt gpurun_out/r2k_big_S24E16.txt gpurun_out/r2k_big_K21.txt gpurun_out/r2k_big_C5.txt gpurun_out/r2k_big_RGG24.txt
