"""Diagnostics for the host-input (e2e) path on C2: per-step wall time split
into process_slices / finish / take_reports. Not a benchmark."""
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
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
for rep in range(6):
    eng.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.process_slices_host_ptr(host.data_ptr(), off)
    t1 = time.perf_counter()
    eng.finish()
    t2 = time.perf_counter()
    eng.take_reports()
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"step {rep}: process {1e3*(t1-t0):.2f} finish {1e3*(t2-t1):.2f} take {1e3*(t3-t2):.2f} "
          f"sync {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms")

# per-batch device spans of one traced host-input run
import numpy as np  # noqa: E402
eng.reset()
eng.trace_ops(True)
torch.cuda.synchronize()
t0 = time.perf_counter()
eng.process_slices_host_ptr(host.data_ptr(), off)
eng.finish()
eng.take_reports()
torch.cuda.synchronize()
print(f"traced run {1e3*(time.perf_counter()-t0):.2f} ms")
io = eng.read_io_trace()
half = len(io) // 2
print("chunk copies done (ms):", np.round(io[:half], 2).tolist())
print("batch launches (ms):   ", np.round(io[half:], 2).tolist())
t = eng.read_op_trace().astype(np.int64)
st, en = t[:, 1], t[:, 2]
base = st.min()
# batches: ops of one launch; a new batch starts where an op starts after the previous op ended
# use slice index: scan ops in order; print every 50th scan op start/end
scans = np.where(t[:, 0] == 0)[0]
for i in range(0, len(scans), 50):
    o = scans[i]
    print(f"scan op {i:4d}: start {(st[o]-base)/1e3:8.1f} us  end {(en[o]-base)/1e3:8.1f} us")
print(f"last op end {(en.max()-base)/1e3:.1f} us")

# host-input run traced: per-op device spans against the copy
eng.reset()
eng.trace_ops(True)
eng.process_slices_host_ptr(host.data_ptr(), off)  # untimed: trace buffers allocate
eng.finish()
eng.take_reports()
eng.reset()
torch.cuda.synchronize()
eng.read_op_trace()
t0 = time.perf_counter()
eng.process_slices_host_ptr(host.data_ptr(), off)
t1 = time.perf_counter()
eng.finish()
eng.take_reports()
t2 = time.perf_counter()
t = eng.read_op_trace().astype(np.int64)
kind, st, en = t[:, 0], t[:, 1], t[:, 2]
base = st.min()
det = np.where(kind == 1)[0]
print(f"traced host-input: process {1e3*(t1-t0):.2f} ms, finish+take {1e3*(t2-t1):.2f} ms, "
      f"kernel span {(en.max()-base)/1e6:.2f} ms, first detect at {(st[det[0]]-base)/1e6:.2f} ms")
ends = en[det]
print("detect period (median, us):", np.median(np.diff(ends)) / 1e3)
for i in (0, 50, 100, 150, 200, 250, 300):
    if i < len(det):
        print(f"  detect {i}: end {(ends[i]-base)/1e6:.3f} ms")
