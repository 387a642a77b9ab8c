#!/bin/bash
# a last randomised parity campaign on the final code (fresh seeds)
OUT=gpurun_out/${TAG:-r02ff}; mkdir -p $OUT
for sd in 121 122 123; do timeout 900 python scripts/fuzz_parity.py 500 $sd > $OUT/fuzz_parity_s$sd.txt 2>&1; echo "fuzz_parity s$sd: $(tail -1 $OUT/fuzz_parity_s$sd.txt)"; done
for sd in 124 125 126; do timeout 1500 python scripts/fuzz_parity.py 120 $sd 6 > $OUT/fuzz_parity_large_s$sd.txt 2>&1; echo "fuzz_parity 6x s$sd: $(tail -1 $OUT/fuzz_parity_large_s$sd.txt)"; done
timeout 900 python scripts/fuzz_more.py 400 127 > $OUT/fuzz_more_s127.txt 2>&1; echo "fuzz_more s86: $(tail -1 $OUT/fuzz_more_s127.txt)"
timeout 900 python scripts/fuzz_kernels.py 300 128 > $OUT/fuzz_kernels_s128.txt 2>&1; echo "fuzz_kernels s87: $(tail -1 $OUT/fuzz_kernels_s128.txt)"
for sd in 129 130; do timeout 900 python scripts/fuzz_ring.py 12 $sd > $OUT/fuzz_ring_s$sd.txt 2>&1; echo "fuzz_ring s$sd: $(tail -1 $OUT/fuzz_ring_s$sd.txt)"; done
grep -h FAIL $OUT/*.txt | head
