"""Compare whole-step CUDA-event timing with the per-launch profile hooks
(measurement helper)."""
import ctypes as C
import numpy as np
import torch
import paper_1005_2314_b200 as pb

cfg = pb.GeneratorConfig(pool_size=4096, discard_every=2, disable_chi2=True)
seeds = np.arange(1, 16385, dtype=np.uint64)
stream = torch.cuda.current_stream()
b = pb.PoolBatch(cfg, n_pools=16384, seeds=seeds, dtype="f32", stream=stream)
b.snapshot()
out = torch.empty((16384, 1 << 18), dtype=torch.float32, device="cuda")
L = pb._capi.load()
for rnd in range(3):
    for _ in range(3):
        b.fill_from_snapshot_into(out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        b.fill_from_snapshot_into(out)
    e1.record(stream)
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 10
    L.wallace_profile_begin(b.h)
    for _ in range(10):
        b.fill_from_snapshot_into(out)
    pm, pn, qm, qn = C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()
    L.wallace_profile_end(b.h, C.byref(pm), C.byref(pn), C.byref(qm), C.byref(qn))
    print(f"round {rnd}: step {step:.4f} ms; profiled pool {pm.value / pn.value:.4f} ms x{pn.value}, "
          f"plan {qm.value / max(1, qn.value) * 1e3:.1f} us x{qn.value}")
