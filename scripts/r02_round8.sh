#!/bin/bash
OUT=gpurun_out/${TAG:-r02o}; mkdir -p $OUT
timeout 900 python scripts/fuzz_parity.py 120 3 6 107 > $OUT/case107.txt 2>&1; echo "case107: $(tail -2 $OUT/case107.txt)"
timeout 1500 python scripts/fuzz_parity.py 120 3 6 > $OUT/fuzz_parity_large_s3.txt 2>&1; echo "fuzz scale6 seed 3: $(tail -1 $OUT/fuzz_parity_large_s3.txt)"
timeout 1500 python scripts/fuzz_parity.py 120 2 6 > $OUT/fuzz_parity_large_s2.txt 2>&1; echo "fuzz scale6 seed 2: $(tail -1 $OUT/fuzz_parity_large_s2.txt)"
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_ring_multirank.py -q -rf > $OUT/t_sr.log 2>&1; echo "stream+ring rc=$? $(tail -1 $OUT/t_sr.log)"
grep -h FAIL $OUT/*.txt | head
