"""Diagnostics for the persistent engine on C2: H2D bandwidth, per-op device
spans (scan / detect) of a device-resident run and of the host-input (e2e)
run. Not a benchmark."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_09246_b200 import abi, native, synth  # noqa: E402

w = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
tr = synth.trace(w)
off = tr.offsets()
total = int(off[-1])
host = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
tr.generate(out=host.numpy().view(abi.PAIR_DTYPE))
d = host.to("cuda", non_blocking=False)
torch.cuda.synchronize()

for nbytes in (64 << 20, total * 8):
    src = host[:nbytes]
    dst = d[:nbytes]
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"H2D {nbytes/1e6:.0f} MB: {nbytes/best/1e6:.1f} GB/s")


def summarize(tag, t):
    if len(t) == 0:
        print(tag, "no ops")
        return
    kind, st, en = t[:, 0], t[:, 1].astype(np.int64), t[:, 2].astype(np.int64)
    span = (en - st) / 1e3
    t0 = st.min()
    tot = (en.max() - t0) / 1e3
    sc, de = kind == 0, kind == 1
    print(f"{tag}: ops={len(t)} total={tot:.0f}us scan n={sc.sum()} sum={span[sc].sum():.0f}us "
          f"mean={span[sc].mean():.2f}us | detect n={de.sum()} sum={span[de].sum():.0f}us "
          f"mean={span[de].mean() if de.any() else 0:.2f}us")
    # gaps between consecutive ops (end of op i to end of op i+1 minus span)
    order = np.argsort(st)
    gaps = (st[order][1:] - en[order][:-1]) / 1e3
    det0 = st[de].min() if de.any() else en.max()
    print(f"   first detect starts at {(det0 - t0)/1e3:.0f}us; after it {(en.max()-det0)/1e3:.0f}us "
          f"= {(en.max()-det0)/1e3/max(1, de.sum()):.2f}us per detected slice")
    print(f"   op gaps: sum={gaps.sum():.0f}us  max={gaps.max():.1f}us  "
          f"(negative = overlap: {gaps[gaps<0].sum():.0f}us)")
    # scans before the first detection vs after
    first_det = np.argmax(de) if de.any() else len(t)
    pre = sc.copy(); pre[first_det:] = False
    post = sc.copy(); post[:first_det] = False
    if pre.any():
        print(f"   scan spans before first detect: mean={span[pre].mean():.2f}us  after: "
              f"mean={span[post].mean() if post.any() else 0:.2f}us")
    return tot


eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
for rep in range(3):
    eng.reset()
    eng.trace_ops(rep == 2)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.process_slices(offsets=off, device_ptr=d.data_ptr())
    eng.finish()
    eng.take_reports()
    torch.cuda.synchronize()
    print(f"device-input run {rep}: {(time.perf_counter()-t)*1e3:.2f} ms wall")
summarize("device-input", eng.read_op_trace())
print("detect diag (traced run)", eng.detect_diag())
eng.trace_ops(False)
print("detect phases", eng.detect_phases())
print("detect latency", eng.detect_latency())
for rep in range(6):
    eng.reset()
    eng.trace_ops(rep == 5)
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.process_slices_host_ptr(host.data_ptr(), off)
    eng.finish()
    eng.take_reports()
    torch.cuda.synchronize()
    print(f"host-input run {rep}: {(time.perf_counter()-t)*1e3:.2f} ms wall")
summarize("host-input", eng.read_op_trace())

# per-CTA view of a detected-slice pair (scan op after a detect, then detect)
eng.reset()
eng.trace_ops(True)
eng.process_slices(offsets=off, device_ptr=d.data_ptr())
eng.finish()
eng.take_reports()
ct = eng.read_cta_trace().astype(np.int64)
tr_ = eng.read_op_trace()
kinds = tr_[-ct.shape[0]:, 0] if len(tr_) else None
print("cta trace", ct.shape)
if kinds is not None:
    names = ["start", "A1", "bar1", "B/A2", "bar2", "C", "epi", "end", "rec", "copies", "reset", "last", "bar0", "touch"]
    for o in range(ct.shape[0] - 6, ct.shape[0] - 2):
        base = ct[o - 1, :, 7].min()
        if kinds[o] == 0:
            st, en = ct[o, :, 0], ct[o, :, 7]
            print(f"op {o} scan: start [{(st.min()-base)/1e3:.1f},{(st.max()-base)/1e3:.1f}] "
                  f"end [{(en.min()-base)/1e3:.1f},{(en.max()-base)/1e3:.1f}]us")
            continue
        row = []
        for j in range(14):
            v = ct[o, :, j]
            v = v[v > 0]
            if len(v):
                row.append(f"{names[j]}=[{(v.min()-base)/1e3:.1f},{np.median(v-base)/1e3:.1f},{(v.max()-base)/1e3:.1f}]")
        print(f"op {o} detect (min,med,max us):", " ".join(row))

# per-CTA phase durations over all detect ops of the traced batch
det = [o for o in range(ct.shape[0]) if kinds is not None and kinds[o] == 1]
if det:
    D = ct[det].astype(np.int64)
    touched = (D[:, :, 13] > 0).any()
    a0 = D[:, :, 13] if touched else D[:, :, 12]
    if touched:
        print("  touch pass per-CTA us: med", np.median((D[:, :, 13] - D[:, :, 12]) / 1e3))
    ph = {"A": D[:, :, 1] - a0, "bar1": D[:, :, 2] - D[:, :, 1].max(1, keepdims=True),
          "B": D[:, :, 3] - D[:, :, 2], "bar2": D[:, :, 4] - D[:, :, 3].max(1, keepdims=True),
          "C": D[:, :, 5] - D[:, :, 4],
          "bar0": D[:, :, 12] - D[:, :, 0].max(1, keepdims=True)}
    for k, v in ph.items():
        v = v / 1e3
        print(f"  {k:5s} per-CTA us: p10={np.percentile(v,10):.2f} med={np.median(v):.2f} "
              f"p90={np.percentile(v,90):.2f} max={v.max():.2f}")
    last = D[:, :, 11]
    m = last > 0
    print("  epilogue (last->epi) us:", np.median((D[:, :, 6][m] - last[m]) / 1e3))
