# round-2 starting point: GPU tests + one bench line per config on the round-1 code
set -x
mkdir -p gpurun_out/r2b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b/pytest_gpu.log
for c in c1 c2 c3 c4 c5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2b/bench_$c.jsonl 2> gpurun_out/r2b/bench_$c.err; done
tail -2 gpurun_out/r2b/pytest_gpu.log
