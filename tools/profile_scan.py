"""K1 (k_scan) alone over slices of the resident C2 trace, one launch per
slice, for ncu --set full captures. Not a benchmark."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1805_09246_b200 import native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--slices", type=int, default=8)
args = ap.parse_args()
w = synth.WORKLOADS[args.workload]
pairs, off = synth.trace(w).generate(0, args.slices)
d = torch.from_numpy(pairs.view("uint8")).cuda()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
for s in range(args.slices):
    a, b = int(off[s]), int(off[s + 1])
    native.update_pairs(eng.rsra(), eng.slea(), device_ptr=d.data_ptr() + 8 * a, n=b - a)
torch.cuda.synchronize()
print("scanned", int(off[args.slices]), "packets")
