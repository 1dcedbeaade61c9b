python -c "from paper_2505_22938_b200 import build as b; assert not b.stale(), \"stale .so\"" || exit 3
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash scripts/gpu_sweep.sh "c1 c2 c5" "IMF_FOOTPRINT=1" "IMF_FOOTPRINT=0"
