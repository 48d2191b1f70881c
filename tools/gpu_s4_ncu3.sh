# session-4: ncu --set full captures (with source) of the TMA line kernel at the C4 / C2 / C3 shapes
# and of the C4 statistics kernel (exported as CSV on the box: the reports exceed the copy-back limit);
# launch list of the default bench line
set -x
D=gpurun_out/s4ncu; mkdir -p $D; rm -f $D/*
for cfg in "128 4096 e4m3 c4" "256 256 e4m3 c2" "512 64 e3m2 c3"; do
  set -- $cfg
  PROF_N=$1 PROF_BATCH=$2 PROF_FMT=$3 MXFFT_FUSED_IMAGE=0 timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:k_mx_lines_tma -s 2 -c 1 -o /tmp/line_$4 -f python tools/prof_case.py fft2 3 > $D/ncu_$4.log 2>&1
  ncu -i /tmp/line_$4.ncu-rep --page raw --csv > $D/line_$4_raw.csv 2>/dev/null
  ncu -i /tmp/line_$4.ncu-rep --page source --csv > $D/line_$4_src.csv 2>/dev/null
done
PROF_N=128 PROF_BATCH=4096 timeout 600 ncu --set full --clock-control none -k regex:k_ps -s 1 -c 1 -o /tmp/stats_c4 -f python tools/prof_case.py stats 3 > $D/ncu_stats.log 2>&1
ncu -i /tmp/stats_c4.ncu-rep --page raw --csv > $D/stats_c4_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $D/launches_c4.csv python bench.py --no-sweep --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_launches.log 2>&1
ls -la $D
