timeout 1800 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/pytest_slow.log 2>&1; echo slow_rc=$?
