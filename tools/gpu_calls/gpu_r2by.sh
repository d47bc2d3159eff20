export TUNE_PIPE=1 TUNE_NWS=11 TUNE_CHS=5,6,8,16 TUNE_STAGES=2,3,4,5,6,8 TUNE_SLOTS=3,2 TUNE_PIECES=126,254
TUNE_GRID="2:4" timeout 1500 python tools/jit_tune.py C2 0.95 > gpurun_out/ringtune_C2.txt 2>&1; echo "c2=$?"
