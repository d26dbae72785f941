"""cfg1 (one pool, N=1024 fp32, d=1, cubic chi2, 2^24 values) through the
latency kernel vs the one-warp throughput kernel: device ms per fill.
Measurement helper."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1005_2314_b200 as pb

cfg = pb.GeneratorConfig(pool_size=1024, discard_every=1)
dt = sys.argv[1] if len(sys.argv) > 1 else "f32"
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["latency", "throughput"]
for mode in modes:
    b = pb.PoolBatch(cfg, n_pools=1, seeds=[1], dtype=dt)
    b.set_kernel_mode(mode)
    out = torch.empty((1, 1 << 24), dtype=torch.float32 if dt == "f32" else torch.float64, device="cuda")
    b.snapshot()
    b.fill_from_snapshot_into(out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); b.fill_from_snapshot_into(out); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(mode, "ms per 2^24 fill:", [round(t, 3) for t in ts], "launches", pb.kernel_launches())
    b.close()
