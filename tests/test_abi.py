"""CPU-side checks of the drop-in boundary: the C ABI library loads, exports
every entry point include/srlg.h declares, its host-only helpers agree with
the oracle, and the device path fails loudly (no CPU fallback) without a
GPU."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1805_09246_b200 import abi, native

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols(header: Path):
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srlg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = native.LIB_PATH
    assert lib.exists(), "libsrlg.so must be built in-tree"
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (srlg_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols(ROOT / "include" / "srlg.h") if s not in exported]
    assert not missing, missing


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_abi_version():
    assert native.lib().srlg_abi_version() == 1


def test_params_helpers_match_oracle(ora):
    for p in [abi.Params(), abi.Params(seed=808), abi.small_params(7), abi.Params(q_prime=21)]:
        rc, sc = native.rsra_config(p), native.slea_config(p)
        orc, osc = ora.configs(p)
        assert bytes(rc) == bytes(orc)
        assert bytes(sc) == bytes(osc)


@pytest.mark.parametrize("bad", [dict(delta=3), dict(eta_prime=1), dict(q=31), dict(r=2),
                                 dict(theta=4), dict(delta_prime=20000), dict(q_prime=0)])
def test_params_validation_mirrors_reference(ora, bad):
    p = abi.Params(**bad)
    with pytest.raises(abi.ConfigError) as e1:
        native.validate(p)
    with pytest.raises(abi.ConfigError) as e2:
        ora.validate(p)
    assert str(e1.value) == str(e2.value)


def test_no_cpu_fallback_without_gpu():
    if native.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(abi.DeviceError):
        native.Rsra(native.rsra_config(abi.Params()))


def test_report_blob_roundtrip(golden_dir):
    r = np.load(golden_dir / "reports.npz")
    blob = r["engine__trace3_k3__seed7"].tobytes()
    reps = abi.parse_blobs(blob)
    assert len(reps) >= 2
    assert all(r.n_rows if hasattr(r, "n_rows") else True for r in reps)
    csv = abi.reports_to_csv(reps)
    assert csv.startswith("window_end_slice,aip,estimate,flags\n")


def test_reports_csv_matches_reference_writer(ref, golden_dir):
    import ctypes as C

    r = np.load(golden_dir / "reports.npz")
    arr = np.ascontiguousarray(r["c2small__engine"])
    blob = arr.tobytes()
    need = ref._csv(arr.ctypes.data, len(arr), None, 0)
    buf = C.create_string_buffer(need)
    ref._csv(arr.ctypes.data, len(arr), C.addressof(buf), need)
    assert abi.reports_to_csv(abi.parse_blobs(blob)) == buf.value.decode()
