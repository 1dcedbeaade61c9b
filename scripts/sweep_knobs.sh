for s in "IMF_RUNMIN=1024" "IMF_RUNMIN=256" "IMF_RUNMIN=64" "IMF_MAXSUMSQ_K=1048576" "IMF_RUNMIN=100000"; do
  env $s python scripts/quick_bench.py c3 | grep "r48\|r64\|r100" | cut -c1-100 | sed "s/^/$s /"
done
