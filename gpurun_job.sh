timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu_rc=$?
timeout 600 python tools/probe_engine.py > gpurun_out/probe.log 2>&1; echo probe_rc=$?
