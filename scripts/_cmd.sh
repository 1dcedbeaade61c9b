python -c "from paper_2505_22938_b200 import build as b; assert not b.stale(), \"stale .so\"" || exit 3
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2

for e in "IMF_STRIPE_EDGE=2 IMF_STRIPE_MID=3" "IMF_STRIPE_EDGE=1 IMF_STRIPE_MID=3" "IMF_STRIPE_EDGE=2 IMF_STRIPE_MID=2" "IMF_STRIPE_EDGE=3 IMF_STRIPE_MID=4" "IMF_STRIPE_EDGE=1 IMF_STRIPE_MID=2"; do echo $e; env $e timeout 300 python scripts/quick_e2e.py 0; done
