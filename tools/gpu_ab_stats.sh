mkdir -p gpurun_out/abs; rm -f gpurun_out/abs/*
libs="paper_2512_04317_b200/_lib/libmxfft_b200.so $(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)"
for c in 128,4096 256,256 512,64 256,1; do
  timeout 300 python tools/ab_stats.py ${c/,/ } $libs
done > gpurun_out/abs/ab.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stats or prescale" > gpurun_out/abs/pytest.log 2>&1; echo rc=$? >> gpurun_out/abs/pytest.log
