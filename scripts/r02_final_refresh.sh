#!/bin/bash
# refresh the committed bench lines / captures after the last routing changes
OUT=gpurun_out/${TAG:-r02final4}; mkdir -p $OUT
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; python -c "import json;d=json.load(open('$OUT/bench_c4.json'));print('C4', d['value']/1e9, d['e2e']['value']/1e9, d['e2e']['walls_ms'], d['clocks'])"
timeout 900 python bench.py --config C4Z --steps 10 --warmup 3 > $OUT/bench_c4z.json 2> $OUT/bench_c4z.err; python -c "import json;d=json.load(open('$OUT/bench_c4z.json'));print('C4Z', d['value']/1e9, d['e2e']['value']/1e9, d['roofline']['avg_launch_ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgd_fast_kernel|sse_async_kernel" -s 4 -c 2 -o $OUT/c4z_full python bench.py --config C4Z --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_c4z.log 2>&1; echo "ncu c4z rc=$?"
timeout 600 python scripts/rank_probe.py 2 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_ring_multirank.py -q 2>&1 | tail -1
