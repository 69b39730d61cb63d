for i in 1 2 3; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_e$i.json 2> gpurun_out/bench_e$i.err; done
echo done
