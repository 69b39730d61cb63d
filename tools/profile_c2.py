"""One engine pass over a slice range of a workload (device-resident input),
for ncu launch lists / --set full captures. Not a benchmark (numbers taken
under a profiler are never bench values)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1805_09246_b200 import native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--slices", type=int, default=320)
ap.add_argument("--no-persistent", action="store_true")
args = ap.parse_args()
w = synth.WORKLOADS[args.workload]
tr = synth.trace(w)
pairs, off = tr.generate(0, args.slices)
d = torch.from_numpy(pairs.view("uint8")).cuda()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
if args.no_persistent:
    eng.set_persistent(False)
eng.process_slices(offsets=off, device_ptr=d.data_ptr())
eng.finish()
print(len(eng.take_reports()), "report bytes")
print("last detection phases (ns):", native.detect_phase_ns(0))
