"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck):
register and bulk emission, all pass types, latency kernel, consumer, defect
consumer, probes, device seeding, write_stream.  Checker-only helper."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1005_2314_b200 as pb  # noqa: E402

seeds = list(range(1, 9))
for fam, mix in ((0, 0), (0, 1), (1, 0), (1, 1)):
    for dtype in ("f32", "f64"):
        for kw in (dict(pool_size=256, discard_every=2), dict(pool_size=512, discard_every=1, disable_chi2=True)):
            b = pb.PoolBatch(pb.GeneratorConfig(transform_family=fam, mixing=mix, **kw), n_pools=len(seeds),
                             seeds=seeds, dtype=dtype)
            for mode in ("throughput", "latency"):
                b.set_kernel_mode(mode)
                b.fill(3 * kw["pool_size"] + 5)
                b.step_pass(3)
                b.next_pool()
            b.set_kernel_mode("throughput")
            b.consume(2 * kw["pool_size"])
b = pb.PoolBatch(pb.GeneratorConfig(pool_size=256), n_pools=4, seeds=[1, 2, 3, 4], dtype="f32")
b.cross_pool_probes(20)
b.pool_defect_stats(5, 3.0)
b.write_stream(os.devnull, 1000, "f32le")
pb.PoolBatch(pb.GeneratorConfig(pool_size=256), n_pools=4, seeds=[1, 2, 3, 4], dtype="f64", device_seed=True).fill(100)
print("sanitize paths ok")
