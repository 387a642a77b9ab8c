#!/bin/bash
OUT=gpurun_out/r02d; mkdir -p $OUT
export BGMF_ENGINE_OPTS=ordered=1
for cfg in C2 C4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ordered_kernel" -s 3 -c 1 \
  -o $OUT/ord_$cfg python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_$cfg.log 2>&1
echo "ncu $cfg rc=$?"
done
