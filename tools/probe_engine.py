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
import libswap  # noqa: E402,F401

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
eng.set_incremental(0 if "--full" in sys.argv else 2 if "--le" in sys.argv else 1)
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
try:
    print("incremental: re-examined blocks (RSRA, SLEA) over the traced run:", eng.inc_stats())
except Exception as ex:  # an older build
    print("no inc stats", ex)
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

# per-CTA view, by role: stream CTAs run scans and phase A (slots 0 start,
# 12 entry barrier passed, 1 phase A done, 7 op end); reconstruction CTAs run
# det_b (0 start, 12 a_done seen, 14 counts, 13 setup, 19 lists copied,
# 15 tables, 16 DFS, 17 inversion, 18 USLE, 11 last known, 6 epilogue done)
eng.reset()
eng.trace_ops(True)
eng.process_slices(offsets=off, device_ptr=d.data_ptr())
eng.finish()
eng.take_reports()
ct = eng.read_cta_trace().astype(np.int64)
tr_ = eng.read_op_trace()
kinds = tr_[-ct.shape[0]:, 0]
det_ops = [o for o in range(ct.shape[0]) if kinds[o] == 1]
scan_ops = [o for o in range(ct.shape[0]) if kinds[o] == 0]
D = ct[det_ops]
stream = D[:, :, 1] > 0            # CTAs that ran phase A
recon = (D[:, :, 14] > 0)          # CTAs that ran det_b counts


def pct(name, v):
    v = np.asarray(v, dtype=np.float64) / 1e3
    if v.size:
        print(f"  {name:22s} us: p10={np.percentile(v,10):7.2f} med={np.median(v):7.2f} "
              f"p90={np.percentile(v,90):7.2f} max={v.max():7.2f}  (n={v.size})")


print("stream CTAs per detect op:")
pct("entry wait+barrier", (D[:, :, 12] - D[:, :, 0])[stream])
pct("  b_done wait", (D[:, :, 20] - D[:, :, 0])[stream])
pct("  entry barrier", (D[:, :, 12] - D[:, :, 20])[stream])
pct("phase A", (D[:, :, 1] - D[:, :, 12])[stream])
inc = stream & (D[:, :, 13] > 0)
if inc.any():
    pct("  RSRA incremental", (D[:, :, 13] - D[:, :, 12])[inc])
    pct("  SLEA sweep", (D[:, :, 1] - D[:, :, 13])[inc])
pct("A -> op end (barrier)", (D[:, :, 7] - D[:, :, 1])[stream])
S = ct[scan_ops]
late = [i for i, o in enumerate(scan_ops) if o > det_ops[0]]
pct("scan op (after 1st det)", (S[late][:, :, 7] - S[late][:, :, 0])[S[late][:, :, 7] > 0])
# per stream CTA: detect op end -> next scan op start, scan op end -> detect op start
nxt = [i for i, o in enumerate(det_ops) if o + 1 < ct.shape[0] and kinds[o + 1] == 0]
if nxt:
    A_ = ct[[det_ops[i] for i in nxt]]
    B_ = ct[[det_ops[i] + 1 for i in nxt]]
    m_ = (A_[:, :, 7] > 0) & (B_[:, :, 0] > 0) & stream[nxt]
    pct("det end -> scan start", (B_[:, :, 0] - A_[:, :, 7])[m_])
prv = [i for i, o in enumerate(det_ops) if o > 0 and kinds[o - 1] == 0]
if prv:
    A_ = ct[[det_ops[i] - 1 for i in prv]]
    B_ = ct[[det_ops[i] for i in prv]]
    m_ = (A_[:, :, 7] > 0) & (B_[:, :, 0] > 0) & stream[prv]
    pct("scan end -> det start", (B_[:, :, 0] - A_[:, :, 7])[m_])
# which stream CTAs end their scan last (the entry barrier waits for them)
if late:
    E_ = S[late][:, :, 7].astype(np.float64)
    E_[E_ <= 0] = np.nan
    last = np.nanargmax(E_, axis=1)
    ids, cnt = np.unique(last, return_counts=True)
    top = sorted(zip(cnt, ids), reverse=True)[:5]
    print("  last CTA to end the scan (CTA: slices):", ", ".join(f"{i}: {c}" for c, i in top),
          f"of {len(last)}; lag behind the median CTA: "
          f"{np.nanmedian(np.nanmax(E_, axis=1) - np.nanmedian(E_, axis=1)) / 1e3:.2f} us")
# slice period: distance between consecutive detect ops' phase-A end (stream rank max)
aend = np.array([D[i][:, 1][stream[i]].max() for i in range(len(det_ops))])
pct("slice period (A end)", np.diff(aend))
print("reconstruction CTAs per detect op:")
for nm, a, b in (("a_done wait", 0, 12), ("counts", 12, 14), ("setup", 14, 13), ("lists copy", 13, 19),
                 ("table build", 19, 15), ("DFS", 15, 16), ("inversion", 16, 17), ("USLE", 17, 18)):
    m = recon & (D[:, :, b] > 0) & (D[:, :, a] > 0)
    pct(nm, (D[:, :, b] - D[:, :, a])[m])
m = D[:, :, 11] > 0
pct("last known -> epi done", (D[:, :, 6] - D[:, :, 11])[m])
pct("A end -> record (latency)", np.array([D[i][:, 6][m[i]].max() for i in range(len(det_ops))]) - aend)
t_start = ct[:, :, 0][ct[:, :, 0] > 0].min()
pre_end = D[0][:, 12][stream[0]].max()
print(f"scan-only prefix ({det_ops[0]} scan ops): phase A of detection 0 starts "
      f"{(pre_end - t_start) / 1e3:.1f} us after the kernel start "
      f"= {(pre_end - t_start) / 1e3 / max(1, det_ops[0]):.2f} us per slice")
