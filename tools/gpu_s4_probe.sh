# session-4 probe run: instruction-rate probes + state check (GPU tests + bench)
set -x
D=gpurun_out/s4; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
./tools/probe/pipes3 > $D/pipes3.txt 2>&1
./tools/probe/mxb_bench > $D/mxb_bench.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench.jsonl 2> $D/bench.err
tail -3 $D/pytest_gpu.log
cat $D/pipes3.txt $D/mxb_bench.txt
