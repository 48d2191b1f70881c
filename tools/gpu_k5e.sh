D=gpurun_out/k5e; mkdir -p $D; rm -rf $D/*
export PROF_N=128 PROF_BATCH=4096
MXFFT_B200_LIB=$PWD/paper_2512_04317_b200/_lib_timing/libmxfft_b200.so timeout 120 python tools/prof_case.py rtk 1 > $D/timing_rtk.log 2>&1
MXFFT_B200_LIB=$PWD/paper_2512_04317_b200/_lib_timing/libmxfft_b200.so MXFFT_FUSED=1 timeout 120 python tools/prof_case.py rt 1 > $D/timing_rt_all_in_one.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_image -s 1 -c 1 -o $D/image_c4 -f python tools/prof_case.py rtk 3 > $D/ncu_image.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file $D/launches_c4.csv python bench.py --no-sweep --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_launches.log 2>&1
