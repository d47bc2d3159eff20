for f in 16 8 4; do for c in 8 6; do for st in 2 3; do
SC_HOST_FIRST=$f SC_HOST_CHUNKS=$c SC_HOST_STREAMS=$st timeout 120 python tools/e2e_chunks.py > gpurun_out/e2e_f${f}_c${c}_s${st}.txt 2>&1
echo "first=$f chunks=$c streams=$st $(tail -1 gpurun_out/e2e_f${f}_c${c}_s${st}.txt)"
done; done; done > gpurun_out/e2e_sweep.txt
