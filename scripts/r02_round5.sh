#!/bin/bash
OUT=gpurun_out/${TAG:-r02i}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_stream.py -q -rf -s -k "out_of_core" > $OUT/t_ooc.log 2>&1; echo "ooc rc=$? $(tail -1 $OUT/t_ooc.log)"; grep "peak" $OUT/t_ooc.log
timeout 2400 python bench.py --config C5 --steps 3 --warmup 2 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_c5.json'));print(d['value']/1e9, d['e2e']['value']/1e9, d['e2e'].get('wall_s'), d['roofline']['h2d_gbs'])")"
grep "\[bgmf\]" $OUT/bench_c5.err | tail -14
