timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash scripts/gpu_sweep.sh "c2 c5" "IMF_QUAD=0" "IMF_QUAD=1 IMF_SEED_ROWS=8" "IMF_QUAD=1 IMF_SEED_ROWS=16" "IMF_QUAD=1 IMF_SEED_ROWS=4"
