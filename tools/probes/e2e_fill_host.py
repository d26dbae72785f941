"""wallace_fill_host timing on the cfg2 job vs a raw 16 GiB D2H into the same
pinned buffer (measurement helper)."""
import time

import numpy as np
import torch

import paper_1005_2314_b200 as pb

n_pools, count = 16384, 1 << 18
b = pb.PoolBatch(pb.GeneratorConfig(pool_size=4096, discard_every=2, disable_chi2=True), n_pools=n_pools,
                 seeds=np.arange(1, n_pools + 1, dtype=np.uint64))
host = torch.empty((n_pools, count), dtype=torch.float32, pin_memory=True)
dev = torch.empty((n_pools, count), dtype=torch.float32, device="cuda")
for k in range(4):
    t = time.perf_counter()
    b.fill_host_ptr(host.data_ptr(), count)
    print(f"fill_host {k}: {time.perf_counter() - t:.3f} s", flush=True)
for k in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    print(f"raw copy {k}: {time.perf_counter() - t:.3f} s", flush=True)
for k in range(2):
    t = time.perf_counter()
    b.fill_host_ptr(host.data_ptr(), count)
    print(f"fill_host again {k}: {time.perf_counter() - t:.3f} s", flush=True)
