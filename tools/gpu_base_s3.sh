# round-2 session-3 baseline: GPU tests, smoke, default bench line, reference arm
set -x
D=gpurun_out/s3base; mkdir -p $D; rm -rf $D/*
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 300 python __graft_entry__.py > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
( time timeout 900 python bench.py > $D/bench.jsonl 2> $D/bench.err ) 2> $D/bench.time
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.jsonl 2> $D/bench_ref.err ) 2> $D/bench_ref.time
tail -2 $D/pytest_gpu.log; cat $D/bench.time
