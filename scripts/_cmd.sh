python -c "from paper_2505_22938_b200 import build as b; assert not b.stale(), \"stale .so\"" || exit 3
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python scripts/quick_bench.py c3 2>&1 | cut -c1-130
for c in "f32 2048 2048 1 48" "f32 1856 1856 1 48" "u16 2048 2048 1 48"; do timeout 120 python scripts/quick_one.py $c; done
