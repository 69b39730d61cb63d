timeout 300 python tools/probe_engine.py > gpurun_out/probe.log 2>&1; echo probe_rc=$?
