# ncu source-level capture of one line pass per config (C3 n=512, C4 n=128, C2 n=256) for
# bank-conflict hunting; only the per-instruction CSVs and raw metrics come back
for cfg in "512 64" "128 4096" "256 256"; do
  set -- $cfg
  PROF_N=$1 PROF_BATCH=$2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mx_lines -s 2 -c 1 \
    -o /tmp/conf_$1 -f python tools/prof_case.py fft2 3 > gpurun_out/ncu_conf_$1.log 2>&1
  ncu -i /tmp/conf_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/conf_$1_src.csv 2>/dev/null
  ncu -i /tmp/conf_$1.ncu-rep --page raw --csv > gpurun_out/conf_$1_raw.csv 2>/dev/null
done
