import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1005_2314_b200 as pb
from paper_1005_2314_b200 import stats
from oracle.oracle import Cfg, OracleGen
n = 256
kw = dict(pool_size=n)
seeds = [9, 10, 11]
for dt in ["f64"]:
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=3, seeds=seeds, dtype=dt)
    b.set_kernel_mode("latency")
    b.fill(100)
    st = b.get_pool(0) if hasattr(b, "get_pool") else None
    o = OracleGen(Cfg(seed=9, **kw), dt)
    o.fill(100)
    print([m for m in dir(b) if not m.startswith("_")])
    try:
        pool = b.pool(0)
        print("pool equal:", np.array_equal(np.asarray(pool[0] if isinstance(pool, tuple) else pool), o.pool()))
    except Exception as e:
        print("pool err", e)
    acc = b.cross_pool_probes(5, stats.default_probes(n))
    print("acc", acc[0][:2])
