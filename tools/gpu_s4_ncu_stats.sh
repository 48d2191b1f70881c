set -x
D=gpurun_out/s4stats; mkdir -p $D; rm -f $D/*
for cfg in "128 4096 c4" "256 256 c2" "512 64 c3"; do
  set -- $cfg
  PROF_N=$1 PROF_BATCH=$2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ps -s 1 -c 1 -o /tmp/stats_$3 -f python tools/prof_case.py stats 3 > $D/ncu_$3.log 2>&1
  ncu -i /tmp/stats_$3.ncu-rep --page source --csv > $D/stats_$3_src.csv 2>/dev/null
  ncu -i /tmp/stats_$3.ncu-rep --page raw --csv > $D/stats_$3_raw.csv 2>/dev/null
done
ls -la $D
