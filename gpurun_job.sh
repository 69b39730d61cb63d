timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo gpu_rc=$?
