import sys
import numpy as np
import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen
N = 4096
count = int(sys.argv[1]) if len(sys.argv) > 1 else 5 * 4095 + 1
b = pb.PoolBatch(pb.GeneratorConfig(pool_size=N, discard_every=2), n_pools=2, seeds=[1, 2], dtype="f32")
b.set_kernel_mode("throughput")
out = b.fill(count).cpu().numpy()
want = OracleGen(Cfg(seed=1, pool_size=N, discard_every=2), "f32").fill(count)
bad = np.nonzero(out[0].view(np.uint32) != want.view(np.uint32))[0]
print("mismatches", bad.size, bad[:16])
