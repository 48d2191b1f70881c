timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines_big -s 1 -c 1 \
  -o /tmp/big -f python tools/prof_big.py 2 > gpurun_out/ncu_big.log 2>&1
ncu -i /tmp/big.ncu-rep --page source --csv --print-source sass > gpurun_out/big_src.csv 2>/dev/null
ncu -i /tmp/big.ncu-rep --page raw --csv > gpurun_out/big_raw.csv 2>/dev/null
