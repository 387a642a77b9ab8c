#!/bin/bash
OUT=gpurun_out/${TAG:-r02e}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ordered.py -x -q -rA > $OUT/ordered_tests.log 2>&1; echo "ordered tests rc=$? $(tail -1 $OUT/ordered_tests.log)"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rf > $OUT/tests_gpu.log 2>&1; echo "gpu tests rc=$? $(tail -1 $OUT/tests_gpu.log)"
timeout 1200 python scripts/fuzz_parity.py 400 1 > $OUT/fuzz_parity_s1.txt 2>&1; echo "fuzz1 $(tail -1 $OUT/fuzz_parity_s1.txt)"
timeout 1500 python scripts/fuzz_parity.py 150 1 6 > $OUT/fuzz_parity_large.txt 2>&1; echo "fuzz6 $(tail -1 $OUT/fuzz_parity_large.txt)"
timeout 900 python scripts/fuzz_more.py 300 101 > $OUT/fuzz_more.txt 2>&1; echo "fuzzmore $(tail -1 $OUT/fuzz_more.txt)"
