for o in -1 0; do echo OMG=$o; IMF_PAIR_OMG=$o timeout 300 python scripts/quick_bench.py c5 2>&1 | cut -c1-100; done
for t in 56 60; do echo TILE=$t; IMF_TILE=$t timeout 300 python scripts/quick_bench.py c5 2>&1 | cut -c1-100; done
