python -c "from paper_2505_22938_b200 import build as b; assert not b.stale(), \"stale .so\"" || exit 3
IMF_K1U16B=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_u16 -s 1 -c 1 -o gpurun_out/prof_u16b -f python scripts/quick_bench.py c2 > /dev/null 2>&1
ls gpurun_out/prof_u16b*
