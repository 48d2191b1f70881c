# one ncu --set full capture (with source counters) of the C2 prescale statistics kernel
set -x
export PROF_N=${PROF_N:-256} PROF_BATCH=${PROF_BATCH:-256}
timeout 120 python tools/prof_case.py stats 3 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ps -s 2 -c 1 \
  -o gpurun_out/stats_${TAG:-c2} -f python tools/prof_case.py stats 3 > gpurun_out/ncu_stats.log 2>&1
