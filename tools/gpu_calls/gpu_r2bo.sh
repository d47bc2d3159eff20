export TUNE_NWS=11 TUNE_CHS=16,32 TUNE_STAGES=2,3 TUNE_SLOTS=2,3 TUNE_PIECES=254,510
t() { TUNE_GRID="$3" timeout 900 python tools/jit_tune.py "T2:$1" "$2" > "gpurun_out/kltune_$1.txt" 2>&1; echo "$1=$?"; }
t GoogLeNet-Inception5a.1 0.95 "1:8,2:8,1:6"
t GoogLeNet-Inception4a.1 0.9 "1:6,2:6,3:6,1:8"
t GoogLeNet-Inception5a.2 0.9 "1:6,2:6,1:8"
t GoogLeNet-Inception4a.2 0.9 "1:3,2:3,3:3,4:3"
