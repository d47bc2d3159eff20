export TUNE_PIPE=1 TUNE_NWS=11,9,7 TUNE_CHS=16,8,32 TUNE_STAGES=2,3 TUNE_SLOTS=3 TUNE_PIECES=254
TUNE_GRID="2:4,1:4,2:2,3:2,4:2,3:3,2:3,5:2" timeout 1500 python tools/jit_tune.py C2 0.95 > gpurun_out/pipetune_C2.txt 2>&1; echo "c2=$?"
TUNE_GRID="2:4,1:4,2:2,1:2,3:2,2:3,1:3" timeout 1500 python tools/jit_tune.py C4a 0.95 > gpurun_out/pipetune_C4a.txt 2>&1; echo "c4a=$?"
