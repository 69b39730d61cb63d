"""Reconstruction pipeline sweep (srlg_engine_set_recon) on a device-resident
workload: ms per step for each (CTAs, groups), reports checked identical.
Diagnostics, not a benchmark."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_09246_b200 import abi, native, synth  # noqa: E402
import libswap  # noqa: E402,F401  (SRLG_TOOLS_LIB: another build)

w = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
confs = [tuple(int(x) for x in c.split("x")) for c in (sys.argv[2:] or ["16x2", "16x4", "24x4"])]
tr = synth.trace(w)
off = tr.offsets()
total = int(off[-1])
host = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
tr.generate(out=host.numpy().view(abi.PAIR_DTYPE))
d = host.to("cuda")
torch.cuda.synchronize()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
ref = None
for rep in range(2):
    for ctas, groups in confs:
        eng.set_recon(ctas, groups)
        ts = []
        for it in range(5):
            eng.reset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            eng.process_slices(offsets=off, device_ptr=d.data_ptr())
            eng.finish()
            b.record()
            out = eng.take_reports()
            torch.cuda.synchronize()
            if it:
                ts.append(a.elapsed_time(b))
        ref = out if ref is None else ref
        lat = eng.detect_latency()[0]
        print(f"recon {ctas:3d} CTAs x {groups} groups: ms/step median {np.median(ts):.3f} "
              f"-> {total / np.median(ts) / 1e3:.0f} Mpps  latency {lat:.1f} us  "
              f"same={out == ref}", flush=True)
