#!/bin/bash
# u_ring routed by the ratings-per-user CV: throughput on C1..C4Z, C4Z full-size parity, tests
for c in C4Z C4 C3 C2 C1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(\"$c\", '%.3f G/s %.3f ms' % (d['value']/1e9, d['ms_per_step']), d['roofline']['avg_launch_ms'])"; done
timeout 900 python -c "
import sys; sys.path.insert(0,'.')
import paper_2304_13724_b200 as bm
from paper_2304_13724_b200 import workloads
from paper_2304_13724_b200.device import Engine, EngineOptions
for name in ('C4Z','C4','C3','C2'):
    w=workloads.CONFIGS[name]; r,c,v=workloads.generate(name)
    e=Engine(EngineOptions()); e.partition(r,c,v,w.n,w.m,w.grid,w.grid)
    import ctypes
    print(name, 'partitioned', e.nnz)
    e.close()
"
timeout 1500 python -m pytest tests/test_gpu_train.py -q -s -k "zipf" -m slow 2>&1 | grep -h "C4Z\|passed\|failed"
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -1
