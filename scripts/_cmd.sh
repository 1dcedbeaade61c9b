mkdir -p gpurun_out
timeout 1200 python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?
