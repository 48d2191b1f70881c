# round-2 evidence run: GPU tests, smoke, the default bench line (C4 headline +
# every config), the reference arm, the ncu launch list of the headline, and
# ncu --set full captures of the dominant kernels (C4 fused image transform,
# C4 statistics, C5 half-row and last-stage kernels)
set -x
D=gpurun_out/final2; mkdir -p $D; rm -rf $D/*
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 300 python __graft_entry__.py > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench.jsonl 2> $D/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.jsonl 2> $D/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $D/launches_c4.csv python bench.py --no-sweep --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_launches.log 2>&1
export PROF_N=128 PROF_BATCH=4096
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_image -s 1 -c 1 -o $D/image_c4 -f python tools/prof_case.py rtk 3 > $D/ncu_image.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ps -s 1 -c 1 -o $D/stats_c4 -f python tools/prof_case.py stats 3 > $D/ncu_stats.log 2>&1
export PROF_N=16384 PROF_BATCH=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mx_lines_big|k_last_stage" -s 2 -c 2 -o $D/c5_split -f python tools/prof_case.py fft2 2 > $D/ncu_c5.log 2>&1
tail -2 $D/pytest_gpu.log
