#!/bin/bash
OUT=gpurun_out/${TAG:-r02u}; mkdir -p $OUT
for c in C4 C4Z C3; do for f in 0 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --engine-opt u_ring=$f 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(\"$c u_ring\", $f, '%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']), d['train_rmse_trace'][-1], d['roofline']['avg_launch_ms'])"; done; done
for f in 0 1; do timeout 900 python bench.py --config C5 --nnz 600000000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --engine-opt u_ring=$f 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(\"C5(600M) u_ring\", $f, '%.3f G/s %.1f ms' % (d['value']/1e9, d['ms_per_step']), d['roofline']['avg_launch_ms'])"; done
BGMF_ENGINE_OPTS=u_ring=1 timeout 900 python scripts/fuzz_parity.py 300 9 > $OUT/fuzz_uring.txt 2>&1; echo "fuzz u_ring: $(tail -1 $OUT/fuzz_uring.txt)"
