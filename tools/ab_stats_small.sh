libs=$(ls paper_2512_04317_b200/_lib_*/libmxfft_b200.so)
for c in "256 1" "256 8" "512 1" "512 4" "128 16" "128 1"; do timeout 200 python tools/ab_stats.py $c $libs; done
