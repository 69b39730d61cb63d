#!/bin/bash
# GPU-box iteration loop: engine parity subset, a short C2 bench, the engine
# probe's per-slice breakdown. Usage: tools/measure.sh [tag]
tag=${1:-m}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_merge_inbox.py -x -q -m "gpu and not slow" > gpurun_out/t_$tag.log 2>&1
tail -2 gpurun_out/t_$tag.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2> /dev/null > gpurun_out/b_$tag.json
python -c "import json; d=json.load(open('gpurun_out/b_$tag.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'R frac', d['roofline']['frac'], 'det us', d['per_slide_estimate_us'])"
timeout 300 python tools/probe_engine.py c2 > gpurun_out/probe_$tag.txt 2>&1
grep -A30 "stream CTAs per detect op" gpurun_out/probe_$tag.txt | grep -v "^ *$"
