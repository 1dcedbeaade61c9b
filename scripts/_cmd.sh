python -c "from paper_2505_22938_b200 import build as b; assert not b.stale(), \"stale .so\"" || exit 3
IMF_GRANK=1 timeout 900 python -m pytest tests -x -q -m gpu -k "c3 or paths or golden" 2>&1 | tail -2
bash scripts/gpu_sweep.sh "c3" "IMF_GRANK=1" "IMF_GRANK=0"
