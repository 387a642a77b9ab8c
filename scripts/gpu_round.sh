#!/bin/bash
# One gpurun call: smoke, GPU tests, bench, ncu launch list + full capture.
# Usage (under gpurun): bash scripts/gpu_round.sh [tag] [what...]
set -u
TAG=${1:-r01}
shift || true
WHAT=${*:-"smoke tests bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
free -g > $OUT/free.txt 2>&1
B="python bench.py"
for w in $WHAT; do
  case $w in
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" ;;
    tests) timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rA > $OUT/tests_gpu.log 2>&1; echo "tests rc=$?" ;;
    slow) timeout 1500 python -m pytest tests -m "slow" -q -rA -s > $OUT/tests_slow.log 2>&1; echo "slow rc=$?" ;;
    bench) timeout 900 $B --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" ;;
    benchx) for f in "--bulk" "--sse-wide"; do timeout 900 $B --steps 10 --warmup 3 $f --no-e2e --no-cpu-baseline >> $OUT/bench_variants.jsonl 2>> $OUT/bench_variants.err; done; echo "benchx rc=$?" ;;
    h2d) timeout 300 python -c "
import torch,time
for mb in (64,256,1024,4096):
    a=torch.empty(mb<<20,dtype=torch.uint8).pin_memory(); b=torch.empty(mb<<20,dtype=torch.uint8,device='cuda')
    b.copy_(a,non_blocking=True); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): b.copy_(a,non_blocking=True)
    e1.record(); torch.cuda.synchronize(); print('h2d',mb,'MB',5*mb/1024/(e0.elapsed_time(e1)/1e3),'GB/s')
    e0.record()
    for _ in range(5): a.copy_(b,non_blocking=True)
    e1.record(); torch.cuda.synchronize(); print('d2h',mb,'MB',5*mb/1024/(e0.elapsed_time(e1)/1e3),'GB/s')
" > $OUT/h2d.txt 2>&1; nvidia-smi -q | grep -iA3 "pcie gen\|link width" >> $OUT/h2d.txt; echo "h2d rc=$?" ;;
    sse) timeout 900 python -m pytest tests/test_gpu_sse.py -q -rA -x > $OUT/tests_sse.log 2>&1; echo "sse rc=$?" ;;
    benchu) timeout 900 $B --steps 10 --warmup 3 --unfused --no-e2e --no-cpu-baseline > $OUT/bench_unfused.json 2> $OUT/bench_unfused.err; echo "benchu rc=$?" ;;
    benchf) timeout 900 $B --steps 10 --warmup 3 --fused --no-e2e --no-cpu-baseline > $OUT/bench_fused.json 2> $OUT/bench_fused.err; echo "benchf rc=$?" ;;
    small)
      for c in C1 C2 C3; do
        for f in "" "--fused" "--unfused"; do
          timeout 600 $B --config $c --steps 20 --warmup 3 $f --no-e2e --no-cpu-baseline >> $OUT/bench_small.jsonl 2>> $OUT/bench_small.err
        done
      done; echo "small rc=$?" ;;
    c5s) timeout 900 $B --config C5 --nnz 200000000 --steps 3 --warmup 3 --budget-gb 0.5 > $OUT/bench_c5_small.json 2> $OUT/bench_c5_small.err; echo "c5s rc=$?" ;;
    c5) timeout 1500 $B --config C5 --steps 3 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$?" ;;
    probe) timeout 300 python scripts/h2d_probe.py > $OUT/h2d_probe.txt 2>&1; echo "probe rc=$?" ;;
    fuzz) # randomised parity sweeps vs the oracle (trainer, baselines, drop-ins, ring)
      timeout 1500 python scripts/fuzz_parity.py 1500 ${FUZZ_SEED:-1} > $OUT/fuzz_parity.txt 2>&1
      timeout 900 python scripts/fuzz_more.py 400 ${FUZZ_SEED:-1} > $OUT/fuzz_more.txt 2>&1
      timeout 900 python scripts/fuzz_kernels.py 500 ${FUZZ_SEED:-1} > $OUT/fuzz_kernels.txt 2>&1
      timeout 1200 python scripts/fuzz_ring.py 10 ${FUZZ_SEED:-1} > $OUT/fuzz_ring.txt 2>&1
      echo "fuzz rc=$?" ;;
    ksweep) timeout 900 python scripts/k_sweep.py > $OUT/k_sweep.txt 2>&1; echo "ksweep rc=$?" ;;
    rank) timeout 600 python scripts/rank_probe.py 2 > $OUT/rank.txt 2>&1; echo "rank rc=$?" ;;
    dist1) BGMF_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > $OUT/bench_dist1.json 2> $OUT/bench_dist1.err; echo "dist1 rc=$?" ;;
    ncuk) # one kernel, full set + source: NCU_K=<regex> NCU_ARGS=<bench args>
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -s ${NCU_S:-4} -c 1 \
        -o $OUT/k_full $B --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${NCU_ARGS:-} > $OUT/ncu_k.log 2>&1
      echo "ncuk rc=$?" ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches.csv $B --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_bench.log 2>&1
      echo "ncu-list rc=$?"
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sgd_fast_kernel|sse_fast_kernel|sse_async_kernel|epoch_fast_kernel" -s 4 -c 2 \
        -o $OUT/sgd_full $B --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_full.log 2>&1
      echo "ncu-full rc=$?" ;;
  esac
done
