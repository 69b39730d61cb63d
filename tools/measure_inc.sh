#!/bin/bash
# GPU box: incremental-tracking parity, A/B, probe breakdown
tag=${1:-inc}
timeout 900 python -m pytest tests/test_incremental.py tests/test_gpu_parity.py -x -q -m "gpu and not slow" -p no:cacheprovider > gpurun_out/t_$tag.log 2>&1
tail -3 gpurun_out/t_$tag.log
timeout 300 python tools/ab_incremental.py c2 3 > gpurun_out/ab_$tag.txt 2>&1; cat gpurun_out/ab_$tag.txt
timeout 300 python tools/probe_engine.py c2 > gpurun_out/probe_$tag.txt 2>&1
grep -A30 "stream CTAs per detect op" gpurun_out/probe_$tag.txt | grep -v "^ *$"
