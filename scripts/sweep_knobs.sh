IMF_K1_BULK=1 timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for s in "IMF_K1_BULK=0" "IMF_K1_BULK=1" "IMF_K1_BULK=0" "IMF_K1_BULK=1"; do
  env $s python scripts/quick_bench.py c1 c2 c5 | cut -c1-90 | sed "s/^/$s /"
done
