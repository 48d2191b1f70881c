# round-end evidence run: GPU tests, smoke, bench lines for every config + the
# reference arm, the ncu launch list of the default bench, and ncu --set full
# captures of the C2 line kernel and the C2 statistics kernel
set -x
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 300 python bench.py > gpurun_out/final/bench_c2.jsonl 2> gpurun_out/final/bench_c2.err
for c in c1 c3 c4 c5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/final/bench_$c.jsonl 2> gpurun_out/final/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.jsonl 2> gpurun_out/final/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final/ncu_launches.log 2>&1
export PROF_N=256 PROF_BATCH=256
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 -o gpurun_out/final/line_c2 -f python tools/prof_case.py fft2 3 > gpurun_out/final/ncu_line.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ps -s 2 -c 1 -o gpurun_out/final/stats_c2 -f python tools/prof_case.py stats 3 > gpurun_out/final/ncu_stats.log 2>&1
tail -2 gpurun_out/final/pytest_gpu.log
