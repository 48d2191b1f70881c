# K5 profiling: per-phase clocks (timing build), ncu --set full of k_mx_image, tests
set -x
mkdir -p gpurun_out/k5b
export PROF_N=128 PROF_BATCH=4096
MXFFT_B200_LIB=$PWD/paper_2512_04317_b200/_lib_timing/libmxfft_b200.so timeout 120 python tools/prof_case.py rt 3 > gpurun_out/k5b/timing.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_image -s 1 -c 1 -o gpurun_out/k5b/image_c4 -f python tools/prof_case.py rt 3 > gpurun_out/k5b/ncu.log 2>&1
timeout 600 python -m pytest tests/test_gpu_r2.py -x -q -k "fused or apply_prescale" > gpurun_out/k5b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k5b/pytest.log
