for s in "IMF_REFINE=1" "IMF_REFINE=3" "IMF_REFINE=1" "IMF_REFINE=3"; do
  env $s python scripts/quick_bench.py c2 c4 c5 | cut -c1-110 | sed "s/^/$s /"
done
