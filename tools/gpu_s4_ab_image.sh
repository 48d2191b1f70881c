mkdir -p gpurun_out/s4ab; 
libs="paper_2512_04317_b200/_lib/libmxfft_b200.so $(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)"
AB_FUSED=1 AB_MODE=2 AB_K=1 timeout 600 python tools/ab_fft2.py 128 4096 $libs > gpurun_out/s4ab/ab_image.txt 2>&1
cat gpurun_out/s4ab/ab_image.txt
