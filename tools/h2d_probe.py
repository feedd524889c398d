"""Host->device bandwidth from pinned memory: one stream vs two vs four (copy engines)."""
import torch, time
n = 2 * 1024**3 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chunk = n // (ns * 8)
        for c in range(ns * 8):
            s = streams[c % ns]
            with torch.cuda.stream(s):
                d[c * chunk:(c + 1) * chunk].copy_(h[c * chunk:(c + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{ns} stream(s): {n * 8 / dt / 1e9:.1f} GB/s")
