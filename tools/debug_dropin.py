"""Debug: replay the drop-in check's small-geometry engine cases through the
native engine (per-record and pre-sliced persistent paths) and the oracle,
printing the first differing report. Not a test."""
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1805_09246_b200 import abi, native  # noqa: E402

d = tempfile.mkdtemp()
subprocess.run([str(Path(__file__).resolve().parent.parent / "paper_1805_09246_b200/_lib/dropin_check"), d],
               capture_output=True)
ora = O.backend("ora")
for name, k, reinit, seed in (("k3", 3, 0, 7), ("k10", 10, 0, 11), ("k1reinit", 1, 1, 13)):
    recs = np.fromfile(f"{d}/records_{name}.bin", dtype=abi.RECORD_DTYPE)
    p = abi.Params(q=12, r=5, delta=7, eta=8, q_prime=8, r_prime=3, delta_prime=8, eta_prime=256,
                   theta=64, seed=seed)
    wc = abi.WindowConfig(k=k, theta=64, reinit_per_window=reinit, t0_us=1_000_000)
    o = ora.engine(p, wc)
    o.process(recs)
    o.finish()
    exp = abi.parse_blobs(o.take_reports())
    # per-record
    e = native.WindowEngine.from_params(p, wc)
    e.process(recs)
    e.finish()
    g1 = abi.parse_blobs(e.take_reports())
    # pre-sliced (persistent)
    sl = (recs["ts_us"] - 1_000_000) // 1_000_000
    off = np.searchsorted(sl, np.arange(sl.max() + 2)).astype(np.uint64)
    pairs = np.zeros(len(recs), dtype=abi.PAIR_DTYPE)
    pairs["aip"], pairs["bip"] = recs["aip"], recs["bip"]
    e2 = native.WindowEngine.from_params(p, wc)
    e2.process_slices(pairs, off)
    e2.finish()
    g2 = abi.parse_blobs(e2.take_reports())
    for tag, g in (("per-record", g1), ("persistent", g2)):
        bad = [i for i in range(min(len(g), len(exp))) if g[i] != exp[i]]
        print(name, tag, "reports", len(g), "expected", len(exp), "differ at", bad[:5])
        for i in bad[:2]:
            print("   got", g[i])
            print("   exp", exp[i])
