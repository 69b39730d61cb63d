"""bench.py's JSON line: the keys the driver and the judge read (task contract:
metric / value / unit / ms_per_step / e2e / roofline / cpu_baseline /
gpu_launches / clocks), on the small C1 workload. The reference arm runs on
the CPU (oracle/_ref, the reference built from its sources); the GPU arm on
cuda:0."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _common(d):
    assert d["metric"] == METRIC
    assert d["unit"] == "Mpps" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["config"]["workload"] == "c1_discrete_1slice_2^20"
    assert d["vs_baseline"] is None


def test_reference_arm_line():
    if not any((ROOT / "oracle" / "_ref").glob("*.so")):
        pytest.skip("oracle/_ref not built (python -c 'import __graft_entry__ as g; g.build()')")
    d = _run("--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "1")
    _common(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "Mpps", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run("--workload", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    _common(d)
    assert "impl" not in d or d["impl"] != "reference"
    assert d["dtype"] == "u32" and d["data"].startswith("synthetic")
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-2
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * (1 << 20)
    assert e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and isinstance(c["reasons"], list)
