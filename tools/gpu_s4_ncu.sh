# session-4: source-level ncu captures of the C4 fused image kernel and the C2 line kernel
set -x
D=gpurun_out/s4ncu; mkdir -p $D; rm -f $D/*
export PROF_N=128 PROF_BATCH=4096
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_image -s 1 -c 1 -o $D/image_c4 -f python tools/prof_case.py rtk 3 > $D/ncu_image.log 2>&1
export PROF_N=256 PROF_BATCH=256
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 -o $D/line_c2 -f python tools/prof_case.py fft2 3 > $D/ncu_c2.log 2>&1
ls -la $D
