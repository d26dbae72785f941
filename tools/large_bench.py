"""Throughput of the HBM-resident large-pool path (measurement helper)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1005_2314_b200 as pb  # noqa: E402

for P, n, d, count in ((16, 1 << 16, 2, 1 << 22), (256, 1 << 16, 2, 1 << 20), (4, 1 << 20, 2, 1 << 24),
                       (1, 1 << 20, 1, 1 << 24)):
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=n, discard_every=d), n_pools=P,
                     seeds=np.arange(1, P + 1, dtype=np.uint64), dtype="f32")
    out = torch.empty((P, count), dtype=torch.float32, device="cuda")
    b.fill_into(out[:, :1024].contiguous())  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    b.fill_into(out)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{P} pools x N=2^{n.bit_length() - 1} fp32 d={d}: {P * count / dt:.3g} variates/s "
          f"({P * count * 4 / dt / 1e9:.1f} GB/s of output)")
