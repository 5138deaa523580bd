timeout 600 python tools/cta_balance.py C2 3 > gpurun_out/r2au_cta_balance_C2.txt 2>&1; cat gpurun_out/r2au_cta_balance_C2.txt
