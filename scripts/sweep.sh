#!/bin/bash
# tuning sweep of K2 seeding/tile knobs on c2 (development aid)
for T in 64 56 48; do for G in 2 4; do for K in 1 2 4; do
  IMF_TILE=$T IMF_SEED_ROWS=$G IMF_SEEDS=$K python scripts/quick_bench.py c2 2>&1 | tail -1
done; done; done
