cd tools/micro
for r in 0.05 0.1; do ./scan_bench2 $r; done > ../../gpurun_out/scan_bench2.txt 2>&1; echo scan=$?
cd ../..
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu0.log 2>&1; echo pytest=$?
