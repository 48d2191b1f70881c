# K5 bring-up: new GPU tests, then the C4 bench with the fused kernel and without
set -x
mkdir -p gpurun_out/k5
timeout 600 python -m pytest tests/test_gpu_r2.py -x -q -k "fused" > gpurun_out/k5/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/k5/pytest_fused.log
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e > gpurun_out/k5/bench_c4_fused.jsonl 2> gpurun_out/k5/bench_c4_fused.err
MXFFT_FUSED=0 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e > gpurun_out/k5/bench_c4_unfused.jsonl 2> gpurun_out/k5/bench_c4_unfused.err
timeout 900 python -m pytest tests/test_gpu_r2.py -q -k "not fused" > gpurun_out/k5/pytest_r2.log 2>&1; echo "rc=$?" >> gpurun_out/k5/pytest_r2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/k5/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/k5/pytest_parity.log
tail -3 gpurun_out/k5/*.log
