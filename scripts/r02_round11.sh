#!/bin/bash
OUT=gpurun_out/${TAG:-r02r}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ordered.py -q -rf -x > $OUT/t_ord.log 2>&1; echo "ordered rc=$? $(tail -1 $OUT/t_ord.log)"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rf > $OUT/tests_gpu.log 2>&1; echo "gpu tests rc=$? $(tail -1 $OUT/tests_gpu.log)"
timeout 900 python ref_suite/run.py exact > $OUT/ref_exact.log 2>&1; echo "ref exact rc=$? $(tail -1 $OUT/ref_exact.log)"
timeout 600 python -c "
import sys,time; sys.path.insert(0,'.')
import paper_2304_13724_b200 as bm
from paper_2304_13724_b200 import workloads
for name in ('C1','C2'):
    w=workloads.CONFIGS[name]; r,c,v=workloads.generate(name); d=bm.RatingsDataset(w.n,w.m,r,c,v)
    cfg=bm.TrainConfig(k=w.k,grid_i=w.grid,grid_j=w.grid,outer_steps=3,alpha=w.alpha,beta=w.beta)
    for ordv in (0,1):
        o=bm.EngineOptions(exact=True, ordered=bool(ordv))
        bm.train_blocked(d,cfg,early_stop=False,options=o)
        t=time.perf_counter(); res=bm.train_blocked(d,cfg,early_stop=False,options=o); dt=time.perf_counter()-t
        print(name,'exact ordered' if ordv else 'exact 1-thread-per-block', '%.1f ms/epoch' % (dt/3*1e3), [s.train_rmse for s in res.trace])
" > $OUT/exact_speed.txt 2>&1; cat $OUT/exact_speed.txt | tail -4
