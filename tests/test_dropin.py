"""The C++ drop-in (include/slidecard/, libslidecard_b200.so): a
reference-style caller (tests/cpp/dropin_check.cpp) built against the drop-in
headers. On the GPU its self-checks must pass and its WindowEngine /
run_distributed report CSVs must equal the CPU oracle's on the same traces."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1805_09246_b200 import abi

LIB = Path(__file__).resolve().parent.parent / "paper_1805_09246_b200" / "_lib"
CHECK = LIB / "dropin_check"

SMALL = dict(q=12, r=5, delta=7, eta=8, q_prime=8, r_prime=3, delta_prime=8, eta_prime=256,
             theta=64)


def test_dropin_library_and_caller_are_built():
    assert (LIB / "libslidecard_b200.so").exists()
    assert CHECK.exists()
    syms = subprocess.run(["nm", "-DC", "--defined-only", str(LIB / "libslidecard_b200.so")],
                          capture_output=True, text=True, check=True).stdout
    for s in ["slidecard::Rsra::update", "slidecard::Slea::estimate", "slidecard::run_detection",
              "slidecard::WindowEngine::process", "slidecard::run_distributed",
              "slidecard::reconstruct_candidates"]:
        assert s in syms, s


@pytest.mark.gpu
def test_dropin_caller_matches_oracle(tmp_path, ora):
    r = subprocess.run([str(CHECK), str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    for name, k, reinit, seed in [("k3", 3, 0, 7), ("k10", 10, 0, 11), ("k1reinit", 1, 1, 13)]:
        recs = np.fromfile(tmp_path / f"records_{name}.bin", dtype=abi.RECORD_DTYPE)
        wc = abi.WindowConfig(k=k, theta=64, t0_us=1_000_000, reinit_per_window=reinit)
        e = ora.engine(abi.Params(**SMALL, seed=seed), wc)
        e.process(recs)
        e.finish()
        expected = abi.reports_to_csv(abi.parse_blobs(e.take_reports()))
        assert (tmp_path / f"engine_{name}.csv").read_text() == expected, name
