"""Pinned D2H / H2D bandwidth on this box (torch copies, CUDA events)."""
import subprocess
import time

import torch

print(subprocess.run("nvidia-smi topo -m; lscpu | head -20; cat /proc/meminfo | head -3",
                     shell=True, capture_output=True, text=True).stdout)
for gb in (1, 4, 16):
    n = gb << 30
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    t = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    ta = time.time() - t
    for rep in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.copy_(d, non_blocking=True)
        e.record()
        e.synchronize()
        d2h = n / s.elapsed_time(e) / 1e6
        s.record()
        d.copy_(h, non_blocking=True)
        e.record()
        e.synchronize()
        h2d = n / s.elapsed_time(e) / 1e6
        print(f"{gb} GB: pin alloc {ta:.2f}s  D2H {d2h:.1f} GB/s  H2D {h2d:.1f} GB/s", flush=True)
    # two streams, halves
    st = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    t = time.time()
    for i in range(2):
        with torch.cuda.stream(st[i]):
            h[i * n // 2:(i + 1) * n // 2].copy_(d[i * n // 2:(i + 1) * n // 2], non_blocking=True)
    torch.cuda.synchronize()
    print(f"{gb} GB: 2-stream D2H {n / (time.time() - t) / 1e9:.1f} GB/s", flush=True)
    del h, d
