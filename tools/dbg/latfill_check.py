# debug helper: latency-geometry fill vs the oracle (first mismatch, states)
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen
for N, d, dt, cnt in [(1024, 1, "f64", 3000), (1024, 1, "f32", 3000), (256, 2, "f64", 1000), (1024, 1, "f64", 1023)]:
    kw = dict(pool_size=N, discard_every=d)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=2, seeds=[5, 6], dtype=dt)
    b.set_kernel_mode("latency")
    out = b.fill(cnt).cpu().numpy()
    for p, s in enumerate([5, 6]):
        o = OracleGen(Cfg(seed=s, **kw), dt)
        want = o.fill(cnt)
        bad = np.nonzero(out[p] != want)[0]
        print(N, d, dt, cnt, "pool", p, "mismatches", len(bad), "first", bad[:5], out[p][bad[:3]] if len(bad) else "", want[bad[:3]] if len(bad) else "")
    b.close()
