#!/bin/bash
# GPU checks of round 2: GPU suite, the reference's own unit tests through the
# drop-in (exact and fast mode), ring sweeps.
OUT=gpurun_out/${TAG:-r02f}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rf > $OUT/tests_gpu.log 2>&1; echo "gpu tests rc=$? $(tail -1 $OUT/tests_gpu.log)"
timeout 900 python ref_suite/run.py exact > $OUT/ref_suite_exact.log 2>&1; echo "ref exact rc=$? $(tail -1 $OUT/ref_suite_exact.log)"
timeout 900 python ref_suite/run.py fast > $OUT/ref_suite_fast.log 2>&1; echo "ref fast rc=$? $(tail -1 $OUT/ref_suite_fast.log)"
[ -n "$RING" ] && { timeout 1200 python scripts/fuzz_ring.py 10 1 > $OUT/fuzz_ring.txt 2>&1; echo "fuzz ring $(tail -1 $OUT/fuzz_ring.txt)"; }
true
