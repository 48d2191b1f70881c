mkdir -p gpurun_out/ab3; rm -f gpurun_out/ab3/*
libs="paper_2512_04317_b200/_lib/libmxfft_b200.so $(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)"
AB_FUSED=1 timeout 300 python tools/ab_fft2.py 128 4096 $libs > gpurun_out/ab3/ab.txt 2>&1
