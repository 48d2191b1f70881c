# round-2 session-5 evidence run: GPU tests, smoke, the default bench line (C4 headline +
# every config), the reference arm, the ncu launch list of the headline, and ncu --set full
# captures (exported as CSV) of the statistics-folding first pass (k_mx_lines_tma<.., ACC>),
# a plain TMA line pass and k_fold_resolve at the C4 / C2 / C3 shapes
set -x
D=gpurun_out/final_s5; mkdir -p $D; rm -rf $D/*
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 300 python __graft_entry__.py > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench.jsonl 2> $D/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.jsonl 2> $D/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $D/launches_c4.csv python bench.py --no-sweep --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_launches.log 2>&1
for cfg in "128 4096 e4m3 c4" "256 256 e4m3 c2" "512 64 e3m2 c3"; do
  set -- $cfg
  # launches of k_mx_lines_tma per round trip: ACC, plain, plain, plain -> index 4 = the 2nd rep's first pass, 5 = its second
  PROF_N=$1 PROF_BATCH=$2 PROF_FMT=$3 MXFFT_FUSED_IMAGE=0 timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:k_mx_lines_tma -s 4 -c 2 -o /tmp/fold_$4 -f python tools/prof_case.py rt 3 > $D/ncu_$4.log 2>&1
  ncu -i /tmp/fold_$4.ncu-rep --page raw --csv > $D/fold_$4_raw.csv 2>/dev/null
  PROF_N=$1 PROF_BATCH=$2 PROF_FMT=$3 MXFFT_FUSED_IMAGE=0 timeout 600 ncu --set full --clock-control none \
    -k regex:k_fold_resolve -s 1 -c 1 -o /tmp/resolve_$4 -f python tools/prof_case.py rt 3 >> $D/ncu_$4.log 2>&1
  ncu -i /tmp/resolve_$4.ncu-rep --page raw --csv > $D/resolve_$4_raw.csv 2>/dev/null
done
ncu -i /tmp/fold_c4.ncu-rep --page source --csv > $D/fold_c4_src.csv 2>/dev/null
tail -2 $D/pytest_gpu.log; cat $D/smoke.log | tail -2; python tools/bench_summary.py $D/bench.jsonl
