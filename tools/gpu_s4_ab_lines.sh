mkdir -p gpurun_out/s4ab
libs="paper_2512_04317_b200/_lib_old/libmxfft_b200.so paper_2512_04317_b200/_lib/libmxfft_b200.so $(ls paper_2512_04317_b200/_lib_[a-np-z]*/libmxfft_b200.so 2>/dev/null)"
for c in 256,256 512,64; do
  timeout 300 python tools/ab_fft2.py ${c/,/ } $libs
done > gpurun_out/s4ab/ab_lines.txt 2>&1
cat gpurun_out/s4ab/ab_lines.txt
