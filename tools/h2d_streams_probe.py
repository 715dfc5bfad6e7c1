"""Host->device bandwidth with 1, 2 and 4 concurrent copy streams (pinned memory)."""
import time
import torch

GB = 4
src = torch.empty(GB * (1 << 27), dtype=torch.uint64, pin_memory=True)  # GB gigabytes
dst = torch.empty_like(src, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = src.chunk(ns)
    dparts = dst.chunk(ns)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s, hp, dp in zip(streams, parts, dparts):
            with torch.cuda.stream(s):
                dp.copy_(hp, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams={ns} H2D {src.numel() * 8 / dt / 1e9:.1f} GB/s", flush=True)
