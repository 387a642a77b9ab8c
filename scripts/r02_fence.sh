#!/bin/bash
# ordered kernels without the per-visit fence.sc: bit-exactness (repeated), speed
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_ordered.py -q -x 2>&1 | tail -1; done
timeout 900 python scripts/ordered_one_epoch.py C4
timeout 900 python scripts/ordered_one_epoch.py C3
timeout 900 python scripts/exact_bench.py C3 C4 2>&1 | tail -4
timeout 600 python ref_suite/run.py fast 2>&1 | tail -1
timeout 900 python scripts/fuzz_parity.py 300 91 > gpurun_out/fuzz_fence.txt 2>&1; tail -1 gpurun_out/fuzz_fence.txt
