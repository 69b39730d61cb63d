"""Regenerate tests/golden/sketch_streams.npz: "SRLG" v1 sketch streams
written by the REFERENCE's own serialize_sketch (sketch_io.cpp:106-134).

Build container only (needs oracle/_ref). For each case the sketch pair is
driven by the same seeded schedule as states.npz (pairs from the reference
Rng(42), update / slide / reinitialize steps); the fixture stores the
schedule and the exact rsra / slea stream bytes.

Usage: python tests/golden/make_golden_sketch.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import oracle as O  # noqa: E402
from paper_1805_09246_b200 import abi  # noqa: E402

SMALL = dict(q=12, r=5, delta=7, eta=8, q_prime=8, r_prime=3, delta_prime=8, eta_prime=256,
             theta=64)
CASES = [
    ("small_seed7", dict(SMALL, seed=7), [(3000, 1), (2000, 1), (4000, 0)]),
    ("small_seed9_reinit", dict(SMALL, seed=9), [(3000, 2), (2500, 1), (100, 0)]),
    ("default_seed1", dict(seed=1), [(1 << 14, 1), (1 << 13, 0)]),
]


def main():
    be = O.backend("ref")
    out = {}
    for name, pkw, schedule in CASES:
        sk = be.sketch(abi.Params(**pkw))
        pool = be.rng_pair_array(42, sum(n for n, _ in schedule))
        off = 0
        for n, op in schedule:
            sk.update(pool[off: off + n])
            off += n
            if op == 1:
                sk.slide()
            elif op == 2:
                sk.reinit()
        out[f"{name}__rsra"] = np.frombuffer(sk.serialize(1), dtype=np.uint8)
        out[f"{name}__slea"] = np.frombuffer(sk.serialize(2), dtype=np.uint8)
        out[f"{name}__schedule"] = np.array(schedule, dtype=np.uint64)
        out[f"{name}__params"] = np.array([pkw.get(k, getattr(abi.Params(), k)) for k in
                                           ("q", "r", "delta", "eta", "q_prime", "r_prime",
                                            "delta_prime", "eta_prime", "theta", "seed")],
                                          dtype=np.uint64)
    np.savez_compressed(HERE / "sketch_streams.npz", **out)
    print("wrote", HERE / "sketch_streams.npz")


if __name__ == "__main__":
    main()
