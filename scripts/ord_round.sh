#!/bin/bash
# ordered-sweep experiments: bit-exactness tests, then C1-C4 epochs per variant
OUT=gpurun_out/${TAG:-r02c}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ordered.py -x -q -rA > $OUT/ordered_tests.log 2>&1; echo "ordered tests rc=$? $(tail -1 $OUT/ordered_tests.log)"
for cfg in ${CFGS:-C1 C2 C3 C4}; do
  for o in ${VARIANTS:-ordered=0 ordered=1,ord_warp=1 ordered=1,ord_warp=0}; do
    f=$OUT/bench_${cfg}_${o//[=,]/_}
    BGMF_ENGINE_OPTS=$o timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $f.json 2> $f.err
    echo "$cfg $o rc=$? $(python -c "import json;d=json.load(open('$f.json'));print('%.3f G/s %.3f ms/ep rmse %.9f' % (d['value']/1e9, d['ms_per_step'], d['train_rmse_trace'][-1]))" 2>&1 | tail -1)"
  done
done
