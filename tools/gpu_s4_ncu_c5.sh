set -x
D=gpurun_out/s4c5; mkdir -p $D; rm -f $D/*
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines_big -s 2 -c 1 -o /tmp/c5_half -f python tools/c5_pass_probe.py > $D/ncu_c5.log 2>&1
ncu -i /tmp/c5_half.ncu-rep --page source --csv > $D/c5_half_src.csv 2>/dev/null
ncu -i /tmp/c5_half.ncu-rep --page raw --csv > $D/c5_half_raw.csv 2>/dev/null
ls -la $D
