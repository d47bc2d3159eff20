TUNE_FULL=1 TUNE_NWS="11,7,4" TUNE_CHS="4,10,20" TUNE_STAGES="2" TUNE_SLOTS="2,3" TUNE_PIECES="126,254" timeout 1500 python tools/jit_tune.py C1 0.9 > gpurun_out/jit_tune_C1.txt 2>&1; echo tune=$?
