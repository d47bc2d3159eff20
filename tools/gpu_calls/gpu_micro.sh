set -x
./tools/micro/interp_bench > gpurun_out/interp_bench.log 2>&1; echo interp=$?
timeout 300 python tools/probe_run.py > gpurun_out/probe.log 2>&1; echo probe=$?
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_sparse.py -x -q -k "test_small_batch_all_outputs and C4b" > gpurun_out/memcheck.log 2>&1; echo memcheck=$?
