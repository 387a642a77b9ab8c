#!/bin/bash
# run-aligned sweep chunk edges (snap = max entries an edge moves): epochs, rank shape, parity
OUT=gpurun_out/${TAG:-r02s}; mkdir -p $OUT
for c in C4 C4Z C3 C2; do for f in ${SN:-0 32 128}; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --engine-opt snap=$f 2>$OUT/err_${c}_$f.txt | python -c "import json,sys;d=json.load(sys.stdin);print(\"$c snap\", $f, '%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']), d['train_rmse_trace'][-1], d['roofline']['avg_launch_ms'])"; done; done
for f in ${SN:-0 32 128}; do echo "rank snap=$f"; BGMF_ENGINE_OPTS=snap=$f timeout 600 python scripts/rank_probe.py 2 2>&1 | grep blocks/launch; done
for f in ${SN5:-0 128}; do timeout 900 python bench.py --config C5 --nnz 600000000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --engine-opt snap=$f 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(\"C5(600M) snap\", $f, '%.3f G/s %.1f ms' % (d['value']/1e9, d['ms_per_step']), d['roofline']['avg_launch_ms'])"; done
BGMF_ENGINE_OPTS=snap=${FS:-128} timeout 900 python scripts/fuzz_parity.py 300 9 > $OUT/fuzz_snap.txt 2>&1; echo "fuzz snap: $(tail -1 $OUT/fuzz_snap.txt)"
