"""The reference's own unit tests (proj/tests/test_{hash, sliding_counters,
linear_counting, rsra, slea, window, distributed, sketch_io, config}.cpp),
compiled UNMODIFIED against the drop-in headers and libslidecard_b200 with a
doctest stand-in (build.py build_ref_unit_tests; tests/cpp/doctest_shim).
Their device-backed cases run on the GPU: every test case must pass there,
i.e. a caller of the reference needs no source change."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "paper_1805_09246_b200" / "_lib" / "ref_unit_tests"


def _run(*args):
    if not BIN.exists():
        pytest.skip("ref_unit_tests not built (needs /root/reference at build time)")
    return subprocess.run([str(BIN), *args], capture_output=True, text=True, timeout=1200)


def test_host_only_cases_pass_without_gpu():
    """cases that never touch a device (hash known answers, counter
    semantics, config validation, linear counting) pass anywhere"""
    r = _run("lsb")
    assert r.returncode == 0, r.stdout + r.stderr
    for name in ("sampling threshold", "le_estimate", "corrected_weight", "defaults match",
                 "validation rejects"):
        r = _run(name)
        assert r.returncode == 0 and " 0 passed" not in r.stdout, (name, r.stdout, r.stderr)


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_drop_in():
    r = _run()
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-8000:]
    assert "| 0 failed" in r.stdout
