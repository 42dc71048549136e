"""Microbenchmark (tools/): pinned D2H bandwidth of 256 MB with 1-8 concurrent streams (the C2 e2e bound)."""
import torch, time
n = 64 * 1024 * 1024  # 256 MB fp32
d = torch.empty(n, device="cuda")
h = torch.empty(n).pin_memory()
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chunk = n // parts
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i * chunk:(i + 1) * chunk].copy_(d[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(parts, "streams", 4 * n / dt / 1e9, "GB/s")
