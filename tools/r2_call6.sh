python paper_1804_03327_b200/build.py 1 > /dev/null 2>&1
timeout 300 python tools/cta_balance.py C2 3 > gpurun_out/r2f_cta_C2.txt 2>&1; cat gpurun_out/r2f_cta_C2.txt
timeout 300 python tools/cta_balance.py C4 1 > gpurun_out/r2f_cta_C4.txt 2>&1; head -30 gpurun_out/r2f_cta_C4.txt
timeout 900 python tools/fig2_sweep.py K21 10 > gpurun_out/r2f_fig2_K21.txt 2>&1; head -16 gpurun_out/r2f_fig2_K21.txt
timeout 900 python tools/fig6_sample.py K21 100 > gpurun_out/r2f_fig6_K21.txt 2>&1; head -14 gpurun_out/r2f_fig6_K21.txt
