timeout 900 python tools/heur_sweep.py C2 > gpurun_out/r2at_heur_C2.txt 2>&1; cat gpurun_out/r2at_heur_C2.txt
timeout 900 python tools/heur_sweep.py K21 > gpurun_out/r2at_heur_K21.txt 2>&1; cat gpurun_out/r2at_heur_K21.txt
