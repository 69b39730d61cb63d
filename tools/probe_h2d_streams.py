import torch
n = 800 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ch = 8 << 20
for nstreams in (1, 2, 3, 1, 2):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for s in (s1, s2): s.wait_stream(torch.cuda.current_stream())
        ss = [torch.cuda.current_stream(), s1, s2][:nstreams]
        for i in range(0, n, ch):
            with torch.cuda.stream(ss[(i // ch) % nstreams]):
                d[i:i+ch].copy_(h[i:i+ch], non_blocking=True)
        for s in ss[1:]: torch.cuda.current_stream().wait_stream(s)
        b.record(); b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(nstreams, "streams:", round(n / best / 1e6, 1), "GB/s")
