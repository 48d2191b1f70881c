# soak of the fold's randomized test over other seeds (GPU): MXFFT_FOLD_SOAK = 1 .. N
N=${1:-20}
for i in $(seq 1 $N); do
  MXFFT_FOLD_SOAK=$i timeout 600 python -m pytest tests/test_gpu_fold.py -q -x -k randomized 2>&1 | tail -1 | sed "s/^/soak $i: /"
done
