# usage: gpu_n.sh VARIANT CFG S TAG
export SC_FORCE_VARIANT=$1
python tools/prof_run.py $2 $3 1 > gpurun_out/plain_$4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gather_fast -c 1 -o gpurun_out/$4 python tools/prof_run.py $2 $3 1 > gpurun_out/ncu_$4.log 2>&1; echo ncu=$?
