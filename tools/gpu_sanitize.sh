# compute-sanitizer over the hot kernels (small shapes)
mkdir -p gpurun_out/san; rm -f gpurun_out/san/*
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san/$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/san/$tool.log
done
tail -3 gpurun_out/san/*.log
