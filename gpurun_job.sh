timeout 900 python -m pytest tests/test_exact.py -x -q > gpurun_out/pytest_exact.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo gpu_rc=$?
