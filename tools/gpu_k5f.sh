D=gpurun_out/k5f; mkdir -p $D; rm -rf $D/*
export PROF_N=128 PROF_BATCH=4096
MXFFT_B200_LIB=$PWD/paper_2512_04317_b200/_lib_timing/libmxfft_b200.so timeout 120 python tools/prof_case.py rtk 1 > $D/timing_rtk.log 2>&1
timeout 600 python -m pytest tests/test_gpu_r2.py -q -x -k "fused" > $D/pytest.log 2>&1; echo rc=$? >> $D/pytest.log
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e > $D/bench.jsonl 2> $D/bench.err
