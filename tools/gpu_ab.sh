mkdir -p gpurun_out/ab; rm -f gpurun_out/ab/*
libs="paper_2512_04317_b200/_lib/libmxfft_b200.so $(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)"
for c in 256,256 128,4096 512,64 16384,1; do
  timeout 300 python tools/ab_fft2.py ${c/,/ } $libs
done > gpurun_out/ab/ab.txt 2>&1
