"""Single-core copy rate from page-locked memory into a reused 16384-double
buffer (the drop-in Generator's fill(16384) inner loop), with the source
cold (8 MiB block) and warm (256 KiB block).  Measurement helper."""
import time
import numpy as np
import torch

for n in (1 << 20, 1 << 15):
    src = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    src[:] = 1.0
    buf = np.empty(16384)
    reps = (1 << 24) // n
    # cold: evict by touching a 256 MiB array between blocks
    big = np.ones(1 << 25)
    t = 0.0
    for r in range(reps):
        big += 1.0 if r % 4 == 0 else 0.0
        t0 = time.perf_counter()
        for i in range(0, n, 16384):
            np.copyto(buf, src[i:i + 16384])
        t += time.perf_counter() - t0
    print(f"block {n:8d} doubles: {(1 << 24) / t:.3e} values/s")
