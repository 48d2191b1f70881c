mkdir -p gpurun_out/split; rm -f gpurun_out/split/*
timeout 900 python -m pytest tests/test_gpu_r2.py -q -x -k "split or c5" > gpurun_out/split/pytest.log 2>&1; echo rc=$? >> gpurun_out/split/pytest.log
timeout 300 python bench.py --config c5 --no-sweep --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/split/bench_c5.jsonl 2> gpurun_out/split/bench_c5.err
timeout 300 python tools/time_big.py 16384 1 > gpurun_out/split/time_big.txt 2>&1
