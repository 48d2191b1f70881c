mkdir -p gpurun_out/s4ab
libs="$(ls paper_2512_04317_b200/_lib_prev/libmxfft_b200.so 2>/dev/null) paper_2512_04317_b200/_lib/libmxfft_b200.so $(ls paper_2512_04317_b200/_lib_[a-oq-z]*/libmxfft_b200.so 2>/dev/null)"
for c in 128,4096 256,256 512,64; do
  timeout 300 python tools/ab_fft2.py ${c/,/ } $libs
done > gpurun_out/s4ab/ab_lines.txt 2>&1
cat gpurun_out/s4ab/ab_lines.txt
