D=gpurun_out/final2b; mkdir -p $D; rm -rf $D/*
export PROF_N=128 PROF_BATCH=4096 MXFFT_FUSED_IMAGE=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 -o $D/line_c4 -f python tools/prof_case.py rtk 3 > $D/ncu_line_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $D/launches_c4.csv python bench.py --no-sweep --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_launches.log 2>&1
