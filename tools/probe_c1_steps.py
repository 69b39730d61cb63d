"""C1 step breakdown: GPU-side (CUDA events on the engine stream) and host
time of reset / process_slices / finish / take_reports. Diagnostics, not a
benchmark (measured: ~20 / 47 / 60 / 18 us GPU-side; the kernel is ~45 us)."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1805_09246_b200 import abi, native, synth
w = synth.WORKLOADS["c1"]
tr = synth.trace(w); off = tr.offsets(); total = int(off[-1])
host = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
tr.generate(out=host.numpy().view(abi.PAIR_DTYPE))
d = host.to("cuda"); torch.cuda.synchronize()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
stream = torch.cuda.ExternalStream(native.device_stream(0), device=0)
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(8):
    e = [E() for _ in range(5)]
    t = [time.perf_counter()]
    e[0].record(stream); eng.reset(); e[1].record(stream); t.append(time.perf_counter())
    eng.process_slices(offsets=off, device_ptr=d.data_ptr()); e[2].record(stream); t.append(time.perf_counter())
    eng.finish(); e[3].record(stream); t.append(time.perf_counter())
    eng.take_reports(); e[4].record(stream); t.append(time.perf_counter())
    e[4].synchronize()
    print("gpu us:", [round(e[i].elapsed_time(e[i+1])*1e3,1) for i in range(4)], "host us:", [round((t[i+1]-t[i])*1e6,1) for i in range(4)])
