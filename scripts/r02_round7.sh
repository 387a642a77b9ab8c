#!/bin/bash
OUT=gpurun_out/${TAG:-r02n}; mkdir -p $OUT
for cfg in C1 C2 C3 C4; do timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err; echo "$cfg $(python -c "import json;d=json.load(open('$OUT/bench_$cfg.json'));print('%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']), d['roofline']['kernel'], d['gpu_launches'])")"; done
timeout 1500 python scripts/fuzz_parity.py 120 1 6 > $OUT/fuzz_parity_large_s1.txt 2>&1; echo "fuzz scale6 seed 1: $(tail -1 $OUT/fuzz_parity_large_s1.txt)"
timeout 1500 python scripts/fuzz_parity.py 120 3 6 > $OUT/fuzz_parity_large_s3.txt 2>&1; echo "fuzz scale6 seed 3: $(tail -1 $OUT/fuzz_parity_large_s3.txt)"
timeout 900 python scripts/fuzz_parity.py 500 4 > $OUT/fuzz_parity_s4.txt 2>&1; echo "fuzz scale1 seed 4: $(tail -1 $OUT/fuzz_parity_s4.txt)"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rf > $OUT/tests_gpu.log 2>&1; echo "gpu tests rc=$? $(tail -1 $OUT/tests_gpu.log)"
grep -h FAIL $OUT/*.txt | head
