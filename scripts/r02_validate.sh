#!/bin/bash
# round-2 final validation: full GPU suite (incl. slow), fuzz with fresh seeds,
# reference suite, smoke
OUT=gpurun_out/${TAG:-r02val}; mkdir -p $OUT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.log)"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rf > $OUT/tests_gpu.log 2>&1; echo "gpu rc=$? $(tail -1 $OUT/tests_gpu.log)"
timeout 2400 python -m pytest tests -m "slow" -q -rA -s > $OUT/tests_slow.log 2>&1; echo "slow rc=$? $(tail -1 $OUT/tests_slow.log)"
timeout 600 python ref_suite/run.py exact > $OUT/ref_exact.log 2>&1; echo "ref exact: $(tail -1 $OUT/ref_exact.log)"
timeout 600 python ref_suite/run.py fast > $OUT/ref_fast.log 2>&1; echo "ref fast: $(tail -1 $OUT/ref_fast.log)"
for sd in ${SEEDS:-11 12}; do timeout 900 python scripts/fuzz_parity.py 500 $sd > $OUT/fuzz_s$sd.txt 2>&1; echo "fuzz s$sd: $(tail -1 $OUT/fuzz_s$sd.txt)"; done
timeout 1500 python scripts/fuzz_parity.py 120 ${LSEED:-13} 6 > $OUT/fuzz_large_s13.txt 2>&1; echo "fuzz 6x s13: $(tail -1 $OUT/fuzz_large_s13.txt)"
timeout 900 python scripts/fuzz_ring.py 12 ${RSEED:-14} > $OUT/fuzz_ring_s14.txt 2>&1; echo "fuzz ring s14: $(tail -1 $OUT/fuzz_ring_s14.txt)"
grep -h FAIL $OUT/*.txt | head
