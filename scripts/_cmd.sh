python -c "from paper_2505_22938_b200 import build as b; assert not b.stale(), \"stale .so\"" || exit 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_f32_bucket_g -s 0 -c 1 -o gpurun_out/prof_kg -f python scripts/quick_one.py f32 2048 2048 1 64 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv python scripts/quick_one.py f32 2048 2048 1 64 1 2>/dev/null | grep -E "k1_|k2_" | cut -c1-250
