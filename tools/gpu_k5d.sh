mkdir -p gpurun_out/k5d; rm -f gpurun_out/k5d/*
export PROF_N=128 PROF_BATCH=4096
MXFFT_B200_LIB=$PWD/paper_2512_04317_b200/_lib_timing/libmxfft_b200.so timeout 120 python tools/prof_case.py fft2 1 > gpurun_out/k5d/timing.log 2>&1
timeout 600 python -m pytest tests/test_gpu_r2.py -x -q -k "fused" > gpurun_out/k5d/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k5d/pytest.log
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e > gpurun_out/k5d/bench_c4.jsonl 2> gpurun_out/k5d/bench_c4.err
