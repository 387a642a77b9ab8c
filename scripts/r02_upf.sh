#!/bin/bash
# U-row L2 prefetch (u_prefetch): epochs on C4 / C4Z / C3 / C5(600M), the ring-rank shape, parity
OUT=gpurun_out/${TAG:-r02p}; mkdir -p $OUT
for c in C4 C4Z C3; do for f in 0 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --engine-opt u_prefetch=$f 2>$OUT/err_${c}_$f.txt | python -c "import json,sys;d=json.load(sys.stdin);print(\"$c upf\", $f, '%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']), d['train_rmse_trace'][-1], d['roofline']['avg_launch_ms'])"; done; done
for f in 0 1; do echo "rank upf=$f"; BGMF_ENGINE_OPTS=u_prefetch=$f timeout 600 python scripts/rank_probe.py 2 2>&1 | grep blocks/launch; done
for f in 0 1; do timeout 900 python bench.py --config C5 --nnz 600000000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --engine-opt u_prefetch=$f 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(\"C5(600M) upf\", $f, '%.3f G/s %.1f ms' % (d['value']/1e9, d['ms_per_step']), d['roofline']['avg_launch_ms'])"; done
BGMF_ENGINE_OPTS=u_prefetch=1 timeout 900 python scripts/fuzz_parity.py 200 9 > $OUT/fuzz_upf.txt 2>&1; echo "fuzz upf: $(tail -1 $OUT/fuzz_upf.txt)"
timeout 300 python -m pytest tests/test_gpu_partition.py -q -k device_values 2>&1 | tail -1
