#!/bin/bash
# dev aid: scripts/libstats.so = the extension built with -DIMF_STATS (refine / bucket statistics)
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -static-global-template-stub=false -DIMF_STATS"
mkdir -p /tmp/imfstats
for f in imf_sort imf_count imf_pair imf_select imf_direct imf_api imf_peak; do
  nvcc $F -c paper_2505_22938_b200/csrc/$f.cu -o /tmp/imfstats/$f.o &
done
wait
nvcc $F -shared -o scripts/libstats.so /tmp/imfstats/*.o -lcudart
