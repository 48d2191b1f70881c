# ncu --set full captures of the line kernel for C2 (n=256) and C3 (n=512), source-level
mkdir -p gpurun_out/prof; rm -f gpurun_out/prof/*
export PROF_N=256 PROF_BATCH=256
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 -o gpurun_out/prof/line_c2 -f python tools/prof_case.py fft2 3 > gpurun_out/prof/ncu_c2.log 2>&1
export PROF_N=512 PROF_BATCH=64 PROF_FMT=e3m2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 -o gpurun_out/prof/line_c3 -f python tools/prof_case.py fft2 3 > gpurun_out/prof/ncu_c3.log 2>&1
