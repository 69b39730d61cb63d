import sys, time
from pathlib import Path
sys.path.insert(0, "/root/repo")
import torch
total = 800_000_000
host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
host.numpy()[:] = 7
dst = torch.empty(total, dtype=torch.uint8, device="cuda")
cs = torch.cuda.Stream()
for chunk in (total, 256 << 20, 64 << 20, 16 << 20, 4 << 20):
    best = 1e9
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            a.record(cs)
            for o in range(0, total, chunk):
                dst[o:o + chunk].copy_(host[o:o + chunk], non_blocking=True)
            b.record(cs)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"chunk {chunk/2**20:7.1f} MiB: {best:.2f} ms = {total/best/1e6:.1f} GB/s")
