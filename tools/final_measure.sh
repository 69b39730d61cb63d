#!/bin/bash
# GPU-box measurement set for a round's final numbers (tag = file suffix):
# GPU suite, ncu DRAM bytes per workload (bench.py's roofline.traffic), bench
# lines C1/C2/C4/C5 + reference arm + 4 virtual merge ranks, ncu launch list
# of the C2 bench, one ncu --set full capture of k_engine on C2.
tag=${1:-final}
o=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_$tag.log 2>&1; tail -2 $o/pytest_$tag.log
timeout 900 python tools/ncu_dram.py c2 c4 c1 c5 > $o/ncu_dram_$tag.log 2>&1; cp profiles/ncu_dram_*.json $o/
python bench.py > $o/bench_c2_$tag.json 2> $o/bench_c2_$tag.err; head -c 300 $o/bench_c2_$tag.json; echo
for w in c1 c4 c5; do python bench.py --workload $w > $o/bench_${w}_$tag.json 2> $o/bench_${w}_$tag.err; done
python bench.py --impl reference > $o/bench_ref_$tag.json 2> $o/bench_ref_$tag.err
python bench.py --virtual 4 --steps 5 --no-cpu-baseline --no-e2e > $o/bench_v4_$tag.json 2> $o/bench_v4_$tag.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/ncu_launches_$tag.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $o/ncu_launches_$tag.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_engine -c 1 -f -o $o/engine_$tag \
  python tools/profile_c2.py --slices 600 > $o/ncu_full_$tag.log 2>&1
python tools/ncu_summary.py $o/engine_$tag.ncu-rep k_engine > $o/ncu_full_summary_$tag.txt 2>&1
timeout 300 python tools/probe_engine.py c2 > $o/probe_c2_$tag.txt 2>&1
timeout 300 python tools/probe_engine.py c4 > $o/probe_c4_$tag.txt 2>&1
ls $o
