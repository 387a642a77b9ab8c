#!/bin/bash
# u_prefetch routing (auto = on when mean run < 6): C5 full (auto vs off), C4 auto, ring shape, parity
OUT=gpurun_out/${TAG:-r02p2}; mkdir -p $OUT
for f in -1 0; do timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --engine-opt u_prefetch=$f > $OUT/c5_$f.json 2>$OUT/c5_$f.err; python -c "import json;d=json.load(open('$OUT/c5_$f.json'));print('C5 upf', $f, '%.3f G/s %.1f ms' % (d['value']/1e9, d['ms_per_step']), 'e2e %.3f' % (d['e2e']['value']/1e9), d['roofline']['avg_launch_ms'])"; done
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('C4 auto', '%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']))"
BGMF_ENGINE_OPTS=u_prefetch=1 timeout 900 python scripts/fuzz_parity.py 300 9 > $OUT/fuzz_upf.txt 2>&1; echo "fuzz upf=1: $(tail -1 $OUT/fuzz_upf.txt)"
BGMF_ENGINE_OPTS=u_prefetch=1 timeout 900 python scripts/fuzz_parity.py 60 17 6 > $OUT/fuzz_upf_large.txt 2>&1; echo "fuzz upf=1 6x: $(tail -1 $OUT/fuzz_upf_large.txt)"
BGMF_ENGINE_OPTS=u_prefetch=1 timeout 900 python scripts/fuzz_ring.py 8 19 > $OUT/fuzz_ring_upf.txt 2>&1; echo "fuzz ring upf=1: $(tail -1 $OUT/fuzz_ring_upf.txt)"
