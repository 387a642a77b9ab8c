"""Can two ranks on ONE GPU exchange CUDA tensors over gloo (batch_isend_irecv,
all_reduce, broadcast)?  If so the ring trainer's world-2 path can run on a
single-GPU box.  Run: torchrun --nproc-per-node 2 scripts/gloo_cuda_probe.py"""
import os

import torch
import torch.distributed as dist

dist.init_process_group("gloo")
r = dist.get_rank()
torch.cuda.set_device(0)
x = torch.full((4,), float(r + 1), device="cuda:0")
y = torch.zeros(4, device="cuda:0")
ops = [dist.P2POp(dist.isend, x, 1 - r), dist.P2POp(dist.irecv, y, 1 - r)]
for w in dist.batch_isend_irecv(ops):
    w.wait()
z = torch.ones(2, device="cuda:0") * (r + 1)
dist.all_reduce(z)
b = torch.full((3,), float(r), device="cuda:0")
dist.broadcast(b, src=1)
print(f"rank {r}: recv {y.tolist()} allreduce {z.tolist()} bcast {b.tolist()}", flush=True)
dist.destroy_process_group()
