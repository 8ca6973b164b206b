"""H2D bandwidth from pinned memory: one copy vs the same bytes split over 2 / 4 streams."""
import time

import torch

n = 900 * 2**20
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4, 1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * part:(i + 1) * part].copy_(src[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{k} stream(s): {n / dt / 1e9:.1f} GB/s", flush=True)
