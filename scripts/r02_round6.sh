#!/bin/bash
OUT=gpurun_out/${TAG:-r02l}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_ring_multirank.py -q -rf -x > $OUT/t_ring.log 2>&1; echo "ring rc=$? $(tail -1 $OUT/t_ring.log)"
timeout 1500 python scripts/fuzz_ring.py 16 7 > $OUT/fuzz_ring.txt 2>&1; echo "fuzz ring $(tail -1 $OUT/fuzz_ring.txt)"; grep -c "budget=[1-9]" $OUT/fuzz_ring.txt
