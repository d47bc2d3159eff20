export TUNE_PIPE=1 TUNE_NWS=11,9,7,4 TUNE_CHS=16,10,8,32 TUNE_STAGES=2,3 TUNE_SLOTS=3 TUNE_PIECES=254
TUNE_GRID="1:1,2:1,3:1,1:2,2:2,1:4" timeout 1500 python tools/jit_tune.py C1 0.9 > gpurun_out/pipetune_C1.txt 2>&1; echo "c1=$?"
export TUNE_NWS=11,9
TUNE_GRID="3:1,2:1,4:1,2:2,3:2,1:4,2:4" timeout 1500 python tools/jit_tune.py C4b 0.95 > gpurun_out/pipetune_C4b.txt 2>&1; echo "c4b=$?"
TUNE_GRID="3:1,2:1,4:1,2:2,3:2,1:4,2:4" timeout 1500 python tools/jit_tune.py C3 channel > gpurun_out/pipetune_C3.txt 2>&1; echo "c3=$?"
