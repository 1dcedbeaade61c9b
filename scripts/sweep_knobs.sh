for s in "IMF_CHUNK_UNIT=0" "IMF_CHUNK_UNIT=1" "IMF_CHUNK_UNIT=1 IMF_SCRATCH_MB=128" "IMF_CHUNK_UNIT=1 IMF_SCRATCH_MB=112" "IMF_CHUNK_UNIT=0"; do
  env $s python scripts/quick_bench.py c2 c4 c5 | cut -c1-110 | sed "s/^/$s /"
done
