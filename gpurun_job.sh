set -x
timeout 900 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/pytest_slow.log 2>&1; echo slow_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -s 250 -c 200 --csv --log-file gpurun_out/launches_c2.csv python tools/profile_c2.py --slices 320 > /dev/null 2>&1; echo launch_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_detect" -s 600 -c 4 -o gpurun_out/prof_r01 python tools/profile_c2.py --slices 320 > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
