for L in _lib_cr1 _lib_cr3 _lib_cr4 _lib_cr1 _lib_cr3 _lib_cr4; do echo $L; MXFFT_B200_LIB=paper_2512_04317_b200/$L/libmxfft_b200.so timeout 300 python tools/cr_time.py 2>&1 | tail -2; done
