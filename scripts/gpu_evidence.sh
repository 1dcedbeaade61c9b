#!/bin/bash
# Round evidence: suite, smoke, every config, bench lines, launch list, ncu captures.
E=gpurun_out/ev; mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $E/gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $E/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1
timeout 900 python scripts/quick_bench.py c1 c2 c3 c4 c5 > $E/configs.jsonl 2> $E/configs.err
timeout 600 python bench.py > $E/bench_c2.json 2> $E/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $E/bench_reference_c2.json 2>> $E/bench.err
timeout 1200 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > $E/bench_c5.json 2>> $E/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $E/launches_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $E/ncu_bench.log 2>&1
cap() {  # cap NAME KREGEX CONFIG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o $E/prof_$1 -f \
      python scripts/one_config.py $3 > $E/ncu_$1.log 2>&1
}
cap k2_c2 k2_ c2
cap k1_c2 k1_ c2
cap k2_c4hex k2_ c4hex
cap k2_c5 k2_ c5
cap k1_c5 k1_ c5
ls -la $E; tail -3 $E/pytest_gpu.log; cat $E/bench_c2.json | cut -c1-400
