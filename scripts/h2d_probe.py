"""PCIe / host-memory probe: pinned, pageable and cudaHostRegister'ed copies."""
import time

import numpy as np
import torch

cudart = torch.cuda.cudart()


def bw(nbytes, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return reps * nbytes / (time.perf_counter() - t) / 1e9


for mb in (256, 1024, 2400):
    n = mb << 20
    host = np.ones(n, np.uint8)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    th = torch.from_numpy(host)
    print(f"{mb} MB pageable h2d {bw(n, lambda: dev.copy_(th)):.1f} GB/s  "
          f"d2h {bw(n, lambda: th.copy_(dev)):.1f} GB/s")
    t = time.perf_counter()
    rc = cudart.cudaHostRegister(host.ctypes.data, n, 0)
    t_reg = time.perf_counter() - t
    print(f"{mb} MB register {t_reg * 1e3:.1f} ms rc={rc}  registered h2d "
          f"{bw(n, lambda: dev.copy_(th, non_blocking=True)):.1f} GB/s  d2h "
          f"{bw(n, lambda: th.copy_(dev, non_blocking=True)):.1f} GB/s")
    t = time.perf_counter()
    cudart.cudaHostUnregister(host.ctypes.data)
    print(f"{mb} MB unregister {(time.perf_counter() - t) * 1e3:.1f} ms")
    t = time.perf_counter()
    a = np.empty(n // 4, np.float32)
    b = a.astype(np.float64)
    print(f"{mb} MB f32->f64 astype {(time.perf_counter() - t) * 1e3:.1f} ms")
