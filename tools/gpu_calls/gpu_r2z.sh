for L in 1 2; do
TUNE_FULL=1 TUNE_N=512 TUNE_GRID="2:4,3:3,2:2,4:2" TUNE_NWS="11" TUNE_CHS="16,24,32" TUNE_STAGES="2" TUNE_SLOTS="3" TUNE_PIECES="254,510" timeout 1500 python tools/jit_tune.py C5.$L 0.95 > gpurun_out/jit_tune_C5_$L.txt 2>&1; echo tune=$?
done
