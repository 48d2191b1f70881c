mkdir -p gpurun_out/s4ab
libs="paper_2512_04317_b200/_lib_prev/libmxfft_b200.so paper_2512_04317_b200/_lib/libmxfft_b200.so"
timeout 600 python tools/ab_fft2.py 16384 1 $libs > gpurun_out/s4ab/ab_c5.txt 2>&1
cat gpurun_out/s4ab/ab_c5.txt
