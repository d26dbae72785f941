"""Raw device->host bandwidth into pinned memory on this box (measurement helper)."""
import torch
for mib in (64, 256, 1024):
    n = mib << 18
    a = torch.empty(n, dtype=torch.float32, device="cuda")
    b = torch.empty(n, dtype=torch.float32, pin_memory=True)
    best = 1e9
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"D2H {mib} MiB: {n * 4 / best / 1e6:.1f} GB/s")
