set -x
D=gpurun_out/s4ncu; mkdir -p $D
export PROF_N=256 PROF_BATCH=256
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 -o $D/line_c2_tma -f python tools/prof_case.py fft2 3 > $D/ncu_c2_tma.log 2>&1
ls -la $D
