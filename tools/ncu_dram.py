"""DRAM traffic of the dominant kernel per workload, for bench.py's
`roofline.traffic`: runs one engine step of the workload under ncu (the
second k_engine launch: the first is a warm-up), reads
dram__bytes_read.sum + dram__bytes_write.sum and writes
profiles/ncu_dram_<workload name>.json.

  python tools/ncu_dram.py c2 c4 ...        (on the GPU box)
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def one_step(name):
    import numpy as np
    import torch

    from paper_1805_09246_b200 import native, synth

    w = synth.WORKLOADS[name]
    tr = synth.trace(w)
    pairs, off = tr.generate()
    d = torch.from_numpy(pairs.view(np.uint8)).cuda()
    torch.cuda.synchronize()
    eng = native.WindowEngine.from_params(w.sketch_params(), w.window_config(t0_us=0))
    for _ in range(2):
        eng.reset()
        eng.process_slices(offsets=off, device_ptr=d.data_ptr())
        eng.finish()
        eng.take_reports()


def capture(name):
    from paper_1805_09246_b200 import synth

    w = synth.WORKLOADS[name]
    out = subprocess.run(
        ["ncu", "--metrics", METRICS, "--clock-control", "none", "-k", "regex:k_engine",
         "--launch-skip", "1", "--launch-count", "1", "--csv", sys.executable, __file__,
         "--run", name], capture_output=True, text=True, cwd=ROOT)
    rows = [r for r in csv.DictReader(io.StringIO(
        "\n".join(l for l in out.stdout.splitlines() if l.startswith('"'))))]
    vals = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows}
    unit = {r["Metric Name"]: r["Metric Unit"] for r in rows}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3,
             "MB": 1e6, "GB": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1,
             "us": 1e3, "ms": 1e6}
    b = sum(vals[m] * scale[unit[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    rec = {"workload": w.name, "kernel": "k_engine", "dram_bytes_per_launch": b,
           "dram_read_bytes": vals["dram__bytes_read.sum"] * scale[unit["dram__bytes_read.sum"]],
           "dram_write_bytes": vals["dram__bytes_write.sum"] * scale[unit["dram__bytes_write.sum"]],
           "gpu_time_ns_under_ncu": vals["gpu__time_duration.sum"]
           * scale[unit["gpu__time_duration.sum"]],
           "command": f"ncu --metrics {METRICS} --clock-control none -k regex:k_engine "
                      f"--launch-skip 1 --launch-count 1 python tools/ncu_dram.py --run {name}"}
    (ROOT / "profiles" / f"ncu_dram_{w.name}.json").write_text(json.dumps(rec, indent=1) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    if sys.argv[1] == "--run":
        one_step(sys.argv[2])
    else:
        for n in sys.argv[1:]:
            capture(n)
