#!/bin/bash
# round-2 measurement set: smoke, C4 bench (value, e2e, roofline, cpu baseline),
# reference arm, world-1 ring bench, ncu launch list + full captures
OUT=gpurun_out/${TAG:-r02final}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.log)"
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_c4.json'));r=d['roofline'];print(d['value']/1e9, d['e2e']['value']/1e9, r['frac'], r['dram_frac'], r['l2_frac'], d['cpu_baseline']['value']/1e6, d['clocks'])")"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$? $(head -c 300 $OUT/bench_ref.json)"
BGMF_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 > $OUT/bench_dist1.json 2> $OUT/bench_dist1.err; echo "dist1 rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_dist1.json'));print(d['value']/1e9, d['e2e']['value']/1e9, d['roofline'])")"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sgd_fast_kernel|sse_async_kernel" -s 4 -c 2 -o $OUT/c4_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
