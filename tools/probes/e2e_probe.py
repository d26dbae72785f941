"""Where the e2e time goes: a plain 16 GiB D2H copy vs wallace_fill_host (measurement helper)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1005_2314_b200 as pb  # noqa: E402

n = 16384 << 18
host = torch.empty(n, dtype=torch.float32, pin_memory=True)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
for k in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"plain 16 GiB D2H: {dt:.4f} s = {n * 4 / dt / 1e9:.1f} GB/s")
del dev
b = pb.PoolBatch(pb.GeneratorConfig(pool_size=4096, discard_every=2, disable_chi2=True), n_pools=16384,
                 seeds=np.arange(1, 16385, dtype=np.uint64))
for k in range(3):
    t = time.perf_counter()
    b.fill_host_ptr(host.data_ptr(), 1 << 18)
    dt = time.perf_counter() - t
    print(f"fill_host 16 GiB: {dt:.4f} s = {n / dt:.3g} values/s")
dev = torch.empty(n, dtype=torch.float32, device="cuda")
for parts, nstreams in ((16, 1), (16, 2), (64, 2), (8, 2)):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    step = n // parts
    for k in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i in range(parts):
            with torch.cuda.stream(ss[i % nstreams]):
                host[i * step:(i + 1) * step].copy_(dev[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"16 GiB D2H as {parts} copies on {nstreams} streams: {dt:.4f} s = {n * 4 / dt / 1e9:.1f} GB/s")
