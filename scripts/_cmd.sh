timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/quick_bench.py c2 2>&1 | cut -c1-150
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1
