"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs in the build container only (it needs oracle/_ref/libslidecard_ref.so,
compiled from /root/reference by oracle/Makefile). The GPU box and the CPU
test suite only read the committed outputs:

  known_answers.json  hash / seed / geometry / formula known answers
  states.npz          u16 distance arrays after seeded update+slide schedules
  reports.npz         report blobs of engine, detection and distributed runs
  reconstruct.json    reconstruct_candidates on random hot lists

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1805_09246_b200 import abi, synth  # noqa: E402

SMALL = dict(q=12, r=5, delta=7, eta=8, q_prime=8, r_prime=3, delta_prime=8, eta_prime=256,
             theta=64)


def small_params(seed):
    return abi.Params(**SMALL, seed=seed)


def random_records(rng_pairs, n, slices, hosts, t0=1_000_000):
    """acceptance.cpp:69-80 style: ts uniform over `slices`, aip in a small
    host set, bip random; time-ordered."""
    a = rng_pairs
    ts = t0 + (a["aip"][:n].astype(np.uint64) % np.uint64(slices * 1_000_000))
    aip = 0x0A000000 + (a["bip"][:n] % hosts)
    bip = a["bip"][n: 2 * n] if len(a) >= 2 * n else a["aip"][:n]
    rec = np.zeros(n, dtype=abi.RECORD_DTYPE)
    rec["ts_us"], rec["aip"], rec["bip"] = ts, aip, bip
    return rec[np.argsort(rec["ts_us"], kind="stable")]


def heavy(rec_t, aip, peers_pairs, t):
    r = np.zeros(len(peers_pairs), dtype=abi.RECORD_DTYPE)
    r["ts_us"] = t
    r["aip"] = aip
    r["bip"] = np.unique(peers_pairs["bip"])[: len(peers_pairs)]
    return r


def trace_cases(be):
    """Deterministic record traces used for engine/distributed fixtures."""
    cases = {}
    for i, (k, slices, n, hosts) in enumerate([(1, 6, 3000, 24), (3, 10, 5000, 32),
                                               (10, 14, 4000, 16), (3, 8, 6000, 48)]):
        pool = be.rng_pair_array(9000 + i, 2 * n + 400)
        rec = random_records(pool, n, slices, hosts)
        # one heavy host (acceptance.cpp:158-162) so reports are non-trivial
        peers = np.unique(pool["bip"][2 * n:])[:200]
        h = np.zeros(len(peers), dtype=abi.RECORD_DTYPE)
        h["ts_us"] = 1_000_000 + 1_000_000 * (i % slices) + 5
        h["aip"] = 0x0A0000AA
        h["bip"] = peers
        rec = np.concatenate([rec, h])
        rec = rec[np.argsort(rec["ts_us"], kind="stable")]
        cases[f"trace{i}_k{k}"] = (rec, k)
    return cases


def main():
    be = O.backend("ref")
    ka = {}
    ka["mix64"] = {str(x): hex(be.mix64(x)) for x in [0, 1, 2, 0xFFFFFFFF, 0x123456789ABCDEF]}
    ka["hash64"] = {f"{k},{s}": hex(be.hash64(k, s)) for k in [0, 1, 4, 100] for s in [1, 808, 5]}
    ka["lsb"] = {str(x): be.lsb(x) for x in [0, 1, 3, 40, 0x80000000]}
    ka["sampling_threshold"] = {f"{t},{e}": be.sampling_threshold(t, e)
                                for t, e in [(1024, 8), (8, 8), (4, 8), (1025, 8), (1, 1), (64, 8)]}
    ka["detection_rho"] = be.detection_rho().hex()
    ka["le_estimate"] = {f"{w},{e}": [be.le_estimate(w, e)[0].hex(), be.le_estimate(w, e)[1]]
                         for w, e in [(0, 16), (10, 16), (16, 16), (8292.0, 16384), (200.5, 16384)]}
    ka["corrected_weight"] = {f"{w},{s},{e}": be.corrected_weight(w, s, e).hex()
                              for w, s, e in [(100, 0.0, 1024), (8292, 0.5, 16384),
                                              (10, 0.5, 16384), (16384, 0.5, 16384),
                                              (300, 0.01234, 16384)]}
    configs = {}
    for name, p in [("default_seed1", abi.Params()), ("default_seed808", abi.Params(seed=808)),
                    ("small_seed7", small_params(7)), ("qprime21", abi.Params(q_prime=21))]:
        rc, sc = be.configs(p)
        configs[name] = dict(
            params=p.as_dict(),
            rsra=dict(q=rc.q, r=rc.r, delta=rc.delta, eta=rc.eta, tau=rc.tau,
                      seed_h1=hex(rc.seed_h1), seed_h2=hex(rc.seed_h2),
                      seed_rhfg0=hex(rc.seed_rhfg0)),
            slea=dict(q=sc.q, r=sc.r, delta=sc.delta, eta=sc.eta, seed_h3=hex(sc.seed_h3),
                      seeds_lh=[hex(sc.seeds_lh[i]) for i in range(sc.r)]))
        sk = be.sketch(p)
        configs[name]["row_length"] = be.slea_row_length(sk.h)
        configs[name]["rsra_cells"] = be.rsra_ncells(sk.h)
        configs[name]["slea_cells"] = be.slea_ncells(sk.h)
        addrs = [0x0A010203, 0x08080808, 0, 0xFFFFFFFF, 0xC0A80101] + \
            [int(x) for x in be.rng_pair_array(5, 8)["aip"]]
        configs[name]["forward"] = {hex(a): [int(c) for c in be.forward(rc.q, rc.r, rc.delta,
                                                                         rc.seed_rhfg0, a)]
                                    for a in addrs}
        configs[name]["lh_column"] = {hex(a): [be.lh_column(sk.h, i, a) for i in range(sc.r)]
                                      for a in addrs}
        configs[name]["invert"] = {hex(a): [int(x) for x in be.invert(
            rc.q, rc.r, rc.delta, rc.seed_rhfg0,
            be.forward(rc.q, rc.r, rc.delta, rc.seed_rhfg0, a))] for a in addrs}
    ka["configs"] = configs
    (HERE / "known_answers.json").write_text(json.dumps(ka, indent=1, sort_keys=True))

    # ---------------------------------------------------------------- states
    states = {}
    for name, p, schedule in [
        ("small_seed7", small_params(7), [(3000, "slide"), (2000, "slide"), (4000, None)]),
        ("small_seed9_reinit", small_params(9), [(3000, "reinit"), (2500, "slide"), (100, None)]),
        ("default_seed1", abi.Params(), [(1 << 16, "slide"), (1 << 15, None)]),
    ]:
        sk = be.sketch(p)
        pool = be.rng_pair_array(42, sum(n for n, _ in schedule))
        off = 0
        for n, op in schedule:
            sk.update(pool[off: off + n])
            off += n
            if op == "slide":
                sk.slide()
            elif op == "reinit":
                sk.reinit()
        rs, le = sk.cells()
        states[f"{name}__rsra"] = rs
        states[f"{name}__slea"] = le
        states[f"{name}__slides"] = np.array([sk.slides], dtype=np.uint64)
        states[f"{name}__schedule"] = np.array([[n, {"slide": 1, "reinit": 2, None: 0}[op]]
                                                for n, op in schedule], dtype=np.uint64)
    np.savez_compressed(HERE / "states.npz", **states)

    # --------------------------------------------------------------- reports
    reps = {}
    for key, (rec, k) in trace_cases(be).items():
        for seed in (7, 11):
            p = small_params(seed)
            wc = abi.WindowConfig(k=k, theta=64, t0_us=1_000_000, reinit_per_window=int(k == 1))
            e = be.engine(p, wc)
            e.process(rec)
            e.finish()
            reps[f"engine__{key}__seed{seed}"] = np.frombuffer(e.take_reports(), dtype=np.uint8)
        reps[f"records__{key}"] = rec.view(np.uint8)
        p = small_params(5)
        wc = abi.WindowConfig(k=k, theta=64, t0_us=1_000_000)
        for policy in range(3):
            blob, st = be.run_distributed(rec, p, wc, 4, policy)
            reps[f"dist__{key}__policy{policy}"] = np.frombuffer(blob, dtype=np.uint8)
    # default geometry, one discrete slice of a C1-style trace (reduced size)
    w = synth.scaled(synth.WORKLOADS["c1"], packets=1 << 18, planted=20, bg_hosts=100_000)
    tr = synth.trace(w)
    pairs, off = tr.generate()
    reps["c1small__input_sha256"] = np.frombuffer(hashlib.sha256(pairs.tobytes()).digest(),
                                                  dtype=np.uint8)
    e = be.engine(w.sketch_params(), w.window_config(t0_us=0))
    e.process_slices(pairs, off)
    e.finish()
    reps["c1small__engine"] = np.frombuffer(e.take_reports(), dtype=np.uint8)
    # default geometry sliding: 12 slices of a C2-style trace, k = 5
    w2 = synth.scaled(synth.WORKLOADS["c2"], packets=1_200_000, n_slices=12, planted_spread=5,
                      planted=30)
    tr2 = synth.trace(w2)
    pairs2, off2 = tr2.generate()
    reps["c2small__input_sha256"] = np.frombuffer(hashlib.sha256(pairs2.tobytes()).digest(),
                                                  dtype=np.uint8)
    e = be.engine(w2.sketch_params(), w2.window_config(k=5, t0_us=0))
    e.process_slices(pairs2, off2)
    e.finish()
    reps["c2small__engine"] = np.frombuffer(e.take_reports(), dtype=np.uint8)
    np.savez_compressed(HERE / "reports.npz", **reps)

    # ----------------------------------------------------------- reconstruct
    rec_cases = []
    pool = be.rng_pair_array(444, 4000)
    idx = 0
    for inst in range(40):
        q, r, delta, seed = (10, 5, 3, 77) if inst % 2 == 0 else (14, 5, 6, 1234)
        hot = [set() for _ in range(r)]
        for p_ in range(int(pool["aip"][idx] % 4)):
            cols = be.forward(q, r, delta, seed, int(pool["bip"][idx + p_]))
            for i in range(r):
                hot[i].add(int(cols[i]))
        idx += 4
        for i in range(r):
            target = 1 + int(pool["aip"][idx] % 10)
            j = 0
            while len(hot[i]) < target:
                hot[i].add(int(pool["bip"][(idx + j) % len(pool)] % (1 << q)))
                j += 1
            idx += 1
        hot = [sorted(h) for h in hot]
        res = be.reconstruct(q, r, delta, seed, hot)
        tiny_cap = be.reconstruct(q, r, delta, seed, hot, tuple_cap=2)
        rec_cases.append(dict(q=q, r=r, delta=delta, seed=seed, hot=hot,
                              addresses=[int(a) for a in res["addresses"]],
                              overflow=res["overflow"], checked=res["tuples_checked"],
                              kept=res["tuples_kept"], overflow_cap2=tiny_cap["overflow"]))
    (HERE / "reconstruct.json").write_text(json.dumps(rec_cases))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
