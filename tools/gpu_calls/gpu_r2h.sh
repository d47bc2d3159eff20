for c in C2 C4a; do
python tools/prof_run.py $c 0.95 2 > gpurun_out/plain_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum --clock-control none -k regex:compact --csv --log-file gpurun_out/compact_launches_$c.csv python tools/prof_run.py $c 0.95 2 > gpurun_out/ncu_$c.log 2>&1; echo ncu_$c=$?
done
