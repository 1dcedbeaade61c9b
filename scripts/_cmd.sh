bash scripts/gpu_sweep.sh "c5" "IMF_PAIR=0" "IMF_SEED_ROWS=4" "IMF_SEED_ROWS=6" "IMF_TILE=52"
