mkdir -p gpurun_out/ab2; rm -f gpurun_out/ab2/*
libs="paper_2512_04317_b200/_lib/libmxfft_b200.so $(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)"
timeout 300 python tools/ab_fft2.py 16384 1 $libs > gpurun_out/ab2/ab.txt 2>&1
