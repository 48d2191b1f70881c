#!/bin/bash
# A/B every paper_2512_04317_b200/_lib_*/ build against each other on the C2/C4/C3 passes
out=${1:-gpurun_out/ab.txt}
libs=$(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)
for c in 256,256 128,4096 512,64 ${AB_EXTRA}; do
  timeout 200 python tools/ab_fft2.py ${c/,/ } $libs
done > $out 2>&1
