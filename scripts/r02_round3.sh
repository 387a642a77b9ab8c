#!/bin/bash
OUT=gpurun_out/${TAG:-r02g}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_train.py -q -rf -k "late_divergence" > $OUT/t_late.log 2>&1; echo "late-div rc=$? $(tail -1 $OUT/t_late.log)"
timeout 600 python scripts/dsmem_probe.py > $OUT/dsmem_probe.txt 2>&1; echo "dsmem rc=$?"; cat $OUT/dsmem_probe.txt
timeout 900 python bench.py --config C4Z --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_c4z.json 2> $OUT/bench_c4z.err; echo "c4z rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_c4z.json'));print(d['value']/1e9, d['ms_per_step'], d['train_rmse_trace'][-1])")"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgd_fast_kernel|sse_async_kernel" -s 4 -c 2 -o $OUT/c4z_full python bench.py --config C4Z --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_c4z.log 2>&1; echo "ncu c4z rc=$?"
timeout 2400 python -m pytest tests -m "slow" -q -rA -s -k "c4_parity or c4_zipf" > $OUT/tests_slow.log 2>&1; echo "slow rc=$? $(grep -E 'max \|d|passed|failed' $OUT/tests_slow.log | tail -4)"
