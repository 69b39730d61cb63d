import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1805_09246_b200 import abi, native, synth
w = synth.WORKLOADS["c1"]
tr = synth.trace(w); off = tr.offsets(); total = int(off[-1])
host = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
tr.generate(out=host.numpy().view(abi.PAIR_DTYPE))
d = host.to("cuda"); torch.cuda.synchronize()
eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
for rep in range(6):
    t0 = time.perf_counter(); eng.reset(); torch.cuda.synchronize(); t1 = time.perf_counter()
    eng.process_slices(offsets=off, device_ptr=d.data_ptr()); t2 = time.perf_counter()
    eng.finish(); t3 = time.perf_counter()
    eng.take_reports(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"reset {1e3*(t1-t0):.2f} process {1e3*(t2-t1):.2f} finish {1e3*(t3-t2):.2f} take {1e3*(t4-t3):.2f} ms")
