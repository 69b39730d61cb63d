"""Debug: hot-column key distribution of the overlap tables at a C2 slide."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_1805_09246_b200 import native, synth  # noqa: E402

w = synth.WORKLOADS["c2"]
pairs, off = synth.trace(w).generate(0, 305)
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
eng.process_slices(pairs, off)
eng.sync()
hot = eng.rsra().extract_hot(300)
q, delta = 17, 5
ov = (1 << (q - delta)) - 1
for L, h in enumerate(hot):
    h = np.asarray(h, dtype=np.uint64)
    keys = h & ov
    u, c = np.unique(keys, return_counts=True)
    bits = 5
    while (1 << bits) < 2 * len(h):
        bits += 1
    slots = ((keys.astype(np.uint64) * 0x9E3779B1) & 0xFFFFFFFF) >> (32 - bits)
    us, cs = np.unique(slots, return_counts=True)
    print(f"row {L}: n={len(h)} distinct keys={len(u)} max dup key={c.max()} "
          f"table bits={bits} distinct slots={len(us)} max per slot={cs.max()}")
    print("   first cols:", [hex(int(x)) for x in h[:12]])
