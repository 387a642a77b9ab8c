#!/bin/bash
# dynamic sweep chunking (dyn_split = D): C4 / C4Z / C3 epochs and a randomised parity sweep
OUT=gpurun_out/${TAG:-r02d}; mkdir -p $OUT
for c in C4 C4Z C3; do for f in ${DS:-1 2 4}; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --engine-opt dyn_split=$f 2>$OUT/err_$c_$f.txt | python -c "import json,sys;d=json.load(sys.stdin);print(\"$c dyn\", $f, '%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']), d['train_rmse_trace'][-1], d['roofline']['avg_launch_ms'])"; done; done
for f in ${DS5:-1 4}; do timeout 900 python bench.py --config C5 --nnz 600000000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --engine-opt dyn_split=$f 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(\"C5(600M) dyn\", $f, '%.3f G/s %.1f ms' % (d['value']/1e9, d['ms_per_step']), d['roofline']['avg_launch_ms'])"; done
BGMF_ENGINE_OPTS=dyn_split=${FD:-4} timeout 900 python scripts/fuzz_parity.py 300 9 > $OUT/fuzz_dyn.txt 2>&1; echo "fuzz dyn: $(tail -1 $OUT/fuzz_dyn.txt)"
