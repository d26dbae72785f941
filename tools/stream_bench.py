"""Throughput of wallace_write_stream (measurement helper)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1005_2314_b200 as pb  # noqa: E402

for label, P, count, dtype, fmt, target in (
        ("cfg2 shape f32le -> /dev/null", 16384, 1 << 18, "f32", "f32le", "/dev/null"),
        ("cfg2 shape f64le -> /dev/null", 16384, 1 << 17, "f32", "f64le", "/dev/null"),
        ("1 pool f64le -> /dev/shm file", 1, 1 << 25, "f64", "f64le", "/dev/shm/wb_stream.bin"),
        ("1 pool text -> /dev/shm file", 1, 1 << 22, "f64", "text", "/dev/shm/wb_stream.txt")):
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=4096 if P > 1 else 1024, discard_every=2 if P > 1 else 1,
                                        disable_chi2=P > 1),
                     n_pools=P, seeds=np.arange(1, P + 1, dtype=np.uint64), dtype=dtype)
    b.write_stream(target, count, fmt)  # warm-up (allocates and pins the staging buffers)
    t = time.perf_counter()
    b.write_stream(target, count, fmt)
    dt = time.perf_counter() - t
    n = P * count
    size = os.path.getsize(target) if target != "/dev/null" else n * (4 if fmt == "f32le" else 8)
    print(f"{label}: {n:.3g} values in {dt:.3f} s = {n / dt:.3g} values/s, {size / dt / 1e9:.2f} GB/s of output")
    if target.startswith("/dev/shm"):
        os.remove(target)
