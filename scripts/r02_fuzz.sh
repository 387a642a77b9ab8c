#!/bin/bash
# randomised parity campaign (flat 1e-3): trainer at scale 1 and 6, several
# seeds; baselines/hooks/early stopping; drop-in kernels
OUT=gpurun_out/${TAG:-r02m}; mkdir -p $OUT
for sd in 1 2 3; do timeout 900 python scripts/fuzz_parity.py 500 $sd > $OUT/fuzz_parity_s$sd.txt 2>&1; echo "fuzz scale1 seed $sd: $(tail -1 $OUT/fuzz_parity_s$sd.txt)"; done
for sd in 1 2; do timeout 1500 python scripts/fuzz_parity.py 120 $sd 6 > $OUT/fuzz_parity_large_s$sd.txt 2>&1; echo "fuzz scale6 seed $sd: $(tail -1 $OUT/fuzz_parity_large_s$sd.txt)"; done
timeout 900 python scripts/fuzz_more.py 400 5 > $OUT/fuzz_more.txt 2>&1; echo "fuzz_more: $(tail -1 $OUT/fuzz_more.txt)"
timeout 600 python scripts/fuzz_kernels.py 300 5 > $OUT/fuzz_kernels.txt 2>&1; echo "fuzz_kernels: $(tail -1 $OUT/fuzz_kernels.txt)"
grep -h FAIL $OUT/*.txt | head -20
