"""Diagnostics: H2D copy rate of the C2 trace alone and while the engine runs
(device input) concurrently. Not a benchmark."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1805_09246_b200 import abi, native, synth  # noqa: E402

w = synth.WORKLOADS["c2"]
tr = synth.trace(w)
off = tr.offsets()
total = int(off[-1])
host = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
tr.generate(out=host.numpy().view(abi.PAIR_DTYPE))
dev_in = host.to("cuda")
dst = torch.empty_like(dev_in)
cs = torch.cuda.Stream()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
chunk = 64 << 20


def copy_chunks():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        a.record(cs)
        for o in range(0, total * 8, chunk):
            dst[o:o + chunk].copy_(host[o:o + chunk], non_blocking=True)
        b.record(cs)
    return a, b


for rep in range(3):
    a, b = copy_chunks()
    b.synchronize()
    print(f"alone: {a.elapsed_time(b):.2f} ms = {total*8/a.elapsed_time(b)/1e6:.1f} GB/s")
for rep in range(3):
    eng.reset()
    torch.cuda.synchronize()
    a, b = copy_chunks()
    t = time.perf_counter()
    eng.process_slices(offsets=off, device_ptr=dev_in.data_ptr())
    eng.finish()
    b.synchronize()
    torch.cuda.synchronize()
    print(f"with engine: copy {a.elapsed_time(b):.2f} ms = {total*8/a.elapsed_time(b)/1e6:.1f} GB/s; "
          f"wall {1e3*(time.perf_counter()-t):.2f} ms")
