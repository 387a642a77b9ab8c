#!/bin/bash
OUT=gpurun_out/${TAG:-r02q}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_ring_multirank.py -q -rf -k "stream" > $OUT/t_stream.log 2>&1; echo "stream rc=$? $(tail -1 $OUT/t_stream.log)"
timeout 2400 python bench.py --config C5 --steps 3 --warmup 2 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_c5.json'));print(d['value']/1e9, d['e2e']['value']/1e9, d['e2e'].get('wall_s'), d['roofline']['h2d_gbs'], d['e2e']['h2d_bytes_per_step'])")"
grep "\[bgmf\]" $OUT/bench_c5.err | grep -v destroy | tail -8
