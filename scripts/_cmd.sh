python -c "from paper_2505_22938_b200 import build as b; assert not b.stale(), \"stale .so\"" || exit 3
timeout 300 python scripts/quick_bench.py c2 c3 c5 | cut -c1-110
