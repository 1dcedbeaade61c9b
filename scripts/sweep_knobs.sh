timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for s in "IMF_COSTLY_FIRST=0" "IMF_COSTLY_FIRST=1" "IMF_COSTLY_FIRST=0" "IMF_COSTLY_FIRST=1"; do
  env $s python scripts/quick_bench.py c2 c4 c5 | cut -c1-110 | sed "s/^/$s /"
done
