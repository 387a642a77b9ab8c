#!/bin/bash
# spread (partial sweep waves dealt evenly over a full wave of CTAs): ring shape, C1..C4, parity
OUT=gpurun_out/${TAG:-r02sp}; mkdir -p $OUT
for f in 0 1; do echo "rank spread=$f"; BGMF_ENGINE_OPTS=spread=$f timeout 600 python scripts/rank_probe.py 2 2>&1 | grep blocks/launch; done
for c in C4 C4Z C3 C2 C1; do for f in 0 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --engine-opt spread=$f 2>$OUT/err_${c}_$f.txt | python -c "import json,sys;d=json.load(sys.stdin);print(\"$c spread\", $f, '%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']), d['train_rmse_trace'][-1], d['roofline']['avg_launch_ms'])"; done; done
timeout 900 python scripts/fuzz_parity.py 300 27 > $OUT/fuzz.txt 2>&1; echo "fuzz spread: $(tail -1 $OUT/fuzz.txt)"
timeout 900 python scripts/fuzz_ring.py 8 29 > $OUT/fuzz_ring.txt 2>&1; echo "fuzz ring spread: $(tail -1 $OUT/fuzz_ring.txt)"
