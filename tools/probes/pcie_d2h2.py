"""Device->host bandwidth strategies for a 16 GiB block on this box
(measurement helper): one copy, pieces over 1-4 streams, piece sizes."""
import time

import torch

GB = 1 << 30
n = 16 * GB // 4
a = torch.empty(n, dtype=torch.float32, device="cuda")
a.fill_(1.0)
t0 = time.time()
b = torch.empty(n, dtype=torch.float32, pin_memory=True)
print(f"pin 16 GiB: {time.time() - t0:.2f} s", flush=True)
b.fill_(0.0)  # touch


def run(piece_mib, nstreams, reps=2):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    piece = piece_mib << 18
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        k = 0
        for o in range(0, n, piece):
            s = streams[k % nstreams]
            with torch.cuda.stream(s):
                b[o:o + piece].copy_(a[o:o + piece], non_blocking=True)
            k += 1
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"piece {piece_mib:5d} MiB x {nstreams} streams: {16 * GB / best / 1e9:.1f} GB/s", flush=True)


for piece, ns in ((16384, 1), (256, 1), (256, 2), (256, 4), (64, 2), (1024, 2), (2048, 2), (4096, 4)):
    run(piece, ns)
