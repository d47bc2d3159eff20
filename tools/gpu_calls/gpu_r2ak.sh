for v in 60 61; do
timeout 300 python tools/tm_probe.py $v C2 0.9 0.95 0.99 > gpurun_out/tm_probe_$v.txt 2>&1; echo probe$v=$?
done
timeout 300 python tools/tm_probe.py 60 C2:512 0.95 0.99 > gpurun_out/tm_probe_60_512.txt 2>&1; echo p=$?
