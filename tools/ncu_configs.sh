# verification on the committed build + ncu summaries of the C3 / C4 line kernels and the C5 big-line kernel
mkdir -p gpurun_out/cfg
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/cfg/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cfg/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/cfg/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/cfg/smoke.log
for cfg in "512 64" "128 4096"; do
  set -- $cfg
  PROF_N=$1 PROF_BATCH=$2 timeout 600 ncu --set full --clock-control none -k regex:k_mx_lines -s 2 -c 1 \
    -o /tmp/cfg_$1 -f python tools/prof_case.py fft2 3 > gpurun_out/cfg/ncu_$1.log 2>&1
  ncu -i /tmp/cfg_$1.ncu-rep --page raw --csv > gpurun_out/cfg/raw_$1.csv 2>/dev/null
done
timeout 900 ncu --set full --clock-control none -k regex:k_mx_lines_big -s 1 -c 1 -o /tmp/cfg_big -f python tools/prof_big.py 2 > gpurun_out/cfg/ncu_big.log 2>&1
ncu -i /tmp/cfg_big.ncu-rep --page raw --csv > gpurun_out/cfg/raw_big.csv 2>/dev/null
