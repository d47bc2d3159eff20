timeout 300 python tools/probe_run.py "$@" > gpurun_out/probe.log 2>&1; echo probe=$?
