# full GPU test suite + smoke
mkdir -p gpurun_out/full; rm -f gpurun_out/full/*
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/full/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/full/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full/smoke.log
nproc > gpurun_out/full/nproc.txt
tail -3 gpurun_out/full/pytest_gpu.log
