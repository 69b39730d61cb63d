"""A/B of the engine's incremental window tracking (srlg_engine_set_incremental)
on a device-resident workload: alternating runs, CUDA-event times per step.
Not a benchmark (bench.py is); a quick check of one change on one box."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_09246_b200 import abi, native, synth  # noqa: E402
import libswap  # noqa: E402,F401  (SRLG_TOOLS_LIB: another build)

w = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
modes = [int(m) for m in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 1, 0]
tr = synth.trace(w)
off = tr.offsets()
total = int(off[-1])
host = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
tr.generate(out=host.numpy().view(abi.PAIR_DTYPE))
d = host.to("cuda")
torch.cuda.synchronize()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
res = {m: [] for m in modes}
blobs = {}
for rep in range(reps):
    for inc in modes:
        eng.set_incremental(inc)
        for it in range(4):
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
                res[inc].append(a.elapsed_time(b))
            blobs[inc] = out
for inc in modes:
    v = np.array(res[inc])
    print(f"incremental mode {inc}: ms/step median {np.median(v):.3f} min {v.min():.3f} "
          f"-> {total / np.median(v) / 1e3:.0f} Mpps")
print("reports identical:", all(blobs[m] == blobs[modes[0]] for m in modes))
import hashlib  # noqa: E402
print("reports sha", hashlib.sha1(repr(blobs[modes[0]]).encode()).hexdigest()[:16])
print("detect latency", eng.detect_latency())
