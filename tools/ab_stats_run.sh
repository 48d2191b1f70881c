#!/bin/bash
# A/B every paper_2512_04317_b200/_lib_*/ build on the prescale statistics of C2/C4/C3
out=${1:-gpurun_out/abs.txt}
libs=$(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)
for c in "256 256" "128 4096" "512 64"; do
  timeout 200 python tools/ab_stats.py $c $libs
done > $out 2>&1
