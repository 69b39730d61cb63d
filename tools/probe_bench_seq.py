"""Diagnostics for bench.py's resident-input sequence on C2: warm-up, the
diagnostic reads, then timed steps split into reset / process / finish / take
with a device-event span per step. Not a benchmark."""
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
dtrace = host.to("cuda:0")
torch.cuda.synchronize()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
stream = torch.cuda.ExternalStream(native.device_stream(0), device=0)
native.profile_enable(0, True)
mode = sys.argv[1] if len(sys.argv) > 1 else "bench"


def step(log):
    t = [time.perf_counter()]
    eng.reset()
    t.append(time.perf_counter())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.process_slices(offsets=off, device_ptr=dtrace.data_ptr())
    e1.record(stream)  # stream order: completes when the engine kernel does
    t.append(time.perf_counter())
    eng.finish()
    t.append(time.perf_counter())
    eng.take_reports()
    t.append(time.perf_counter())
    e1.synchronize()
    if log:
        d = [round(1e3 * (b - a), 2) for a, b in zip(t, t[1:])]
        print(f"  reset {d[0]} process {d[1]} finish {d[2]} take {d[3]} | device "
              f"{e0.elapsed_time(e1):.2f} ms", flush=True)


for i in range(3):
    print(f"warmup {i}")
    step(True)
if mode == "bench":
    native.profile_read(0)
    native.profile_read_engine(0)
    eng.detect_latency()
    native.kernel_launches()
torch.cuda.synchronize()
if mode == "sleep":
    time.sleep(0.05)
if mode == "nvml":
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
import numpy as np  # noqa: E402
eng.trace_ops(mode == "trace")
for i in range(8):
    print(f"timed {i}")
    step(True)
    t = eng.read_op_trace().astype(np.int64)
    if len(t):
        st, en = t[:, 1], t[:, 2]
        base = st.min()
        dur = en - st
        gaps = st[1:] - en[:-1]
        k = int(np.argmax(dur))
        g = int(np.argmax(gaps)) if len(gaps) else 0
        print(f"  ops {len(t)} span {(en.max()-base)/1e3:.1f} us; longest op #{k} kind {t[k,0]} "
              f"{dur[k]/1e3:.1f} us at {(st[k]-base)/1e3:.1f}; max gap {gaps[g]/1e3:.1f} us "
              f"after op {g}; first op start->first end {(en[0]-st[0])/1e3:.1f} us")
