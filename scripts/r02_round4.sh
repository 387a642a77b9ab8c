#!/bin/bash
OUT=gpurun_out/${TAG:-r02h}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_ordered.py -q -rf > $OUT/t_stream.log 2>&1; echo "stream+ordered rc=$? $(tail -1 $OUT/t_stream.log)"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rf > $OUT/tests_gpu.log 2>&1; echo "gpu tests rc=$? $(tail -1 $OUT/tests_gpu.log)"
timeout 900 python bench.py --config C5 --nnz 200000000 --steps 3 --warmup 2 --budget-gb 0.5 > $OUT/bench_c5s.json 2> $OUT/bench_c5s.err; echo "c5s rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_c5s.json'));print(d['value']/1e9, d['e2e']['value']/1e9, d['e2e'].get('wall_s'))")"
grep "ooc\|partition\|e2e\|epoch" $OUT/bench_c5s.err | tail -20
