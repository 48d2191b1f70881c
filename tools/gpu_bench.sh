# the default bench line (C4 headline + every config) and the reference arm
mkdir -p gpurun_out/bench; rm -f gpurun_out/bench/*
( time timeout 900 python bench.py ) > gpurun_out/bench/bench.jsonl 2> gpurun_out/bench/bench.err
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 3 ) > gpurun_out/bench/ref.jsonl 2> gpurun_out/bench/ref.err
tail -4 gpurun_out/bench/bench.err
