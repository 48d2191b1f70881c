# one ncu --set full capture (with source counters) of the C2 fft2 line kernel
set -x
export PROF_N=${PROF_N:-256} PROF_BATCH=${PROF_BATCH:-256}
timeout 120 python tools/prof_case.py fft2 3 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 \
  -o gpurun_out/line_${TAG:-c2} -f python tools/prof_case.py fft2 3 > gpurun_out/ncu_line.log 2>&1
