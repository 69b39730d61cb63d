"""Pins the CPU checker (oracle/srlg_oracle.c) before anything is compared
against it: golden fixtures generated from the reference library
(tests/golden/make_golden.py), the reference's own frozen numbers
(proj/tests/*.cpp), SURVEY.md Appendix A, and — when oracle/_ref is built —
the reference itself on random inputs."""
import json

import numpy as np
import pytest

from paper_1805_09246_b200 import abi


@pytest.fixture(scope="module")
def ka(golden_dir):
    return json.loads((golden_dir / "known_answers.json").read_text())


@pytest.fixture(scope="module")
def states(golden_dir):
    return np.load(golden_dir / "states.npz")


@pytest.fixture(scope="module")
def reports(golden_dir):
    return np.load(golden_dir / "reports.npz")


def _backends(request):
    return request.param


BACKENDS = ["ora", "ref"]


@pytest.fixture(params=BACKENDS)
def be(request):
    from oracle import oracle as O

    if not O.available(request.param):
        pytest.skip(f"{request.param} not built")
    return O.backend(request.param)


def test_appendix_a_known_answers(ora):
    # SURVEY.md Appendix A (values produced by the built reference)
    assert ora.mix64(0) == 0
    assert ora.mix64(1) == 0x5692161D100B05E5
    assert ora.hash64(1, 1) == 0xBFEF8030DDC2D772
    rc, sc = ora.configs(abi.Params())
    assert (rc.seed_h1, rc.seed_h2, sc.seed_h3, rc.seed_rhfg0) == (
        0xBFEF8030DDC2D772, 0x5F552CE482F2AA47, 0x70335FC3DAF3D8A7, 0xF440FE3B62C79D2C)
    assert sc.seeds_lh[0] == 0xD9973B333AED1A0F and sc.seeds_lh[4] == 0x23C27A5A68B9198A
    assert rc.tau == 7
    a = 0x0A010203
    assert list(ora.forward(17, 5, 5, rc.seed_rhfg0, a)) == [8556, 10620, 41260, 13678, 8652]
    sk = ora.sketch(abi.Params())
    assert [ora.lh_column(sk.h, i, a) for i in range(5)] == [62170, 130700, 31285, 79175, 42240]


def test_reference_frozen_numbers(ora):
    # test_hash.cpp:13-27, test_sliding_counters.cpp:64-77,
    # test_linear_counting.cpp:14-43, test_slea.cpp:35-48
    assert [ora.lsb(x) for x in (3, 40, 1, 0, 0x80000000)] == [0, 3, 0, 32, 31]
    assert [ora.sampling_threshold(t, e) for t, e in
            [(1024, 8), (8, 8), (4, 8), (1025, 8), (1, 1)]] == [7, 0, 0, 8, 0]
    assert abs(ora.detection_rho() - 0.280634) < 1e-6
    assert abs(ora.le_estimate(10, 16)[0] - 15.6933) < 1e-3
    assert ora.le_estimate(16, 16)[1] is True
    assert abs(ora.corrected_weight(8292, 0.5, 16384) - 200.0) < 1e-9
    assert ora.corrected_weight(10, 0.5, 16384) == 0.0
    with pytest.raises(abi.SaturationError):
        ora.corrected_weight(100, 1.0, 1024)
    sk = ora.sketch(abi.Params())
    assert ora.slea_row_length(sk.h) == 2_113_520
    uncovered, covers = ora.group_info(17, 5, 5, 1)
    assert uncovered == 0x1F and covers
    assert not ora.group_info(10, 5, 3, 1)[1]


def test_known_answers_golden(be, ka):
    for x, v in ka["mix64"].items():
        assert be.mix64(int(x)) == int(v, 16)
    for key, v in ka["hash64"].items():
        k, s = map(int, key.split(","))
        assert be.hash64(k, s) == int(v, 16)
    for x, v in ka["lsb"].items():
        assert be.lsb(int(x)) == v
    for key, v in ka["sampling_threshold"].items():
        t, e = map(int, key.split(","))
        assert be.sampling_threshold(t, e) == v
    assert be.detection_rho().hex() == ka["detection_rho"]
    for key, (v, sat) in ka["le_estimate"].items():
        w, e = key.split(",")
        got = be.le_estimate(float(w), int(e))
        assert got[0].hex() == v and got[1] == sat
    for key, v in ka["corrected_weight"].items():
        w, s, e = key.split(",")
        assert be.corrected_weight(float(w), float(s), int(e)).hex() == v


def test_configs_golden(be, ka):
    for name, c in ka["configs"].items():
        p = abi.Params(**c["params"])
        rc, sc = be.configs(p)
        assert rc.tau == c["rsra"]["tau"]
        assert hex(rc.seed_h1) == c["rsra"]["seed_h1"]
        assert hex(rc.seed_h2) == c["rsra"]["seed_h2"]
        assert hex(rc.seed_rhfg0) == c["rsra"]["seed_rhfg0"]
        assert hex(sc.seed_h3) == c["slea"]["seed_h3"]
        assert [hex(sc.seeds_lh[i]) for i in range(sc.r)] == c["slea"]["seeds_lh"]
        sk = be.sketch(p)
        assert be.slea_row_length(sk.h) == c["row_length"]
        assert be.rsra_ncells(sk.h) == c["rsra_cells"]
        for a, cols in c["forward"].items():
            assert list(be.forward(rc.q, rc.r, rc.delta, rc.seed_rhfg0, int(a, 16))) == cols
        for a, cols in c["lh_column"].items():
            assert [be.lh_column(sk.h, i, int(a, 16)) for i in range(sc.r)] == cols
        for a, addrs in c["invert"].items():
            cols = be.forward(rc.q, rc.r, rc.delta, rc.seed_rhfg0, int(a, 16))
            assert list(be.invert(rc.q, rc.r, rc.delta, rc.seed_rhfg0, cols)) == addrs


def _replay_state(be, params, schedule):
    sk = be.sketch(params)
    pool = be.rng_pair_array(42, int(schedule[:, 0].sum()))
    off = 0
    for n, op in schedule:
        sk.update(pool[off: off + int(n)])
        off += int(n)
        if op == 1:
            sk.slide()
        elif op == 2:
            sk.reinit()
    return sk


@pytest.mark.parametrize("name,params", [
    ("small_seed7", abi.small_params(7)),
    ("small_seed9_reinit", abi.small_params(9)),
    ("default_seed1", abi.Params()),
])
def test_states_golden(be, states, name, params):
    sk = _replay_state(be, params, states[f"{name}__schedule"])
    rs, le = sk.cells()
    assert np.array_equal(rs, states[f"{name}__rsra"])
    assert np.array_equal(le, states[f"{name}__slea"])
    assert sk.slides == int(states[f"{name}__slides"][0])


def _records(reports, key):
    return reports[f"records__{key}"].view(abi.RECORD_DTYPE)


@pytest.mark.parametrize("key,k", [("trace0_k1", 1), ("trace1_k3", 3), ("trace2_k10", 10),
                                   ("trace3_k3", 3)])
@pytest.mark.parametrize("seed", [7, 11])
def test_engine_reports_golden(be, reports, key, k, seed):
    rec = _records(reports, key)
    wc = abi.WindowConfig(k=k, theta=64, t0_us=1_000_000, reinit_per_window=int(k == 1))
    e = be.engine(abi.small_params(seed), wc)
    e.process(rec)
    e.finish()
    assert e.take_reports() == reports[f"engine__{key}__seed{seed}"].tobytes()


@pytest.mark.parametrize("key,k", [("trace1_k3", 3), ("trace3_k3", 3)])
@pytest.mark.parametrize("policy", [0, 1, 2])
def test_distributed_golden(be, reports, key, k, policy):
    rec = _records(reports, key)
    wc = abi.WindowConfig(k=k, theta=64, t0_us=1_000_000)
    blob, st = be.run_distributed(rec, abi.small_params(5), wc, 4, policy)
    assert blob == reports[f"dist__{key}__policy{policy}"].tobytes()
    assert st["slice_merges"] > 0 and st["bytes_exchanged"] > 0


def test_full_geometry_reports_golden(be, reports):
    import hashlib

    from paper_1805_09246_b200 import synth

    w = synth.scaled(synth.WORKLOADS["c1"], packets=1 << 18, planted=20, bg_hosts=100_000)
    pairs, off = synth.trace(w).generate()
    assert hashlib.sha256(pairs.tobytes()).digest() == reports["c1small__input_sha256"].tobytes()
    e = be.engine(w.sketch_params(), w.window_config(t0_us=0))
    e.process_slices(pairs, off)
    e.finish()
    got = e.take_reports()
    assert got == reports["c1small__engine"].tobytes()
    reps = abi.parse_blobs(got)
    # all 20 planted supers (2048..4096 distinct peers) are detected
    planted = {a for a, _ in synth.trace(w).planted()}
    assert planted <= {aip for aip, _, _ in reps[0].entries}


def test_reconstruct_golden(be, golden_dir):
    cases = json.loads((golden_dir / "reconstruct.json").read_text())
    for c in cases:
        res = be.reconstruct(c["q"], c["r"], c["delta"], c["seed"], c["hot"])
        assert list(res["addresses"]) == c["addresses"]
        assert res["overflow"] == c["overflow"]
        assert res["tuples_checked"] == c["checked"]
        assert res["tuples_kept"] == c["kept"]
        assert be.reconstruct(c["q"], c["r"], c["delta"], c["seed"], c["hot"],
                              tuple_cap=2)["overflow"] == c["overflow_cap2"]


def test_reconstruct_equals_brute_force(ora):
    # acceptance.cpp:275-328: incremental reconstruction == brute-force
    # enumeration of every tuple through invert
    import itertools

    rng = ora.rng_pair_array(4444, 2000)
    q, r, delta, seed = 10, 5, 3, 77
    for inst in range(30):
        hot = [set() for _ in range(r)]
        for p in range(int(rng["aip"][inst] % 4)):
            cols = ora.forward(q, r, delta, seed, int(rng["bip"][inst * 7 + p]))
            for i in range(r):
                hot[i].add(int(cols[i]))
        for i in range(r):
            j = 0
            while len(hot[i]) < 1 + int(rng["aip"][(inst * 13 + i) % 2000] % 6):
                hot[i].add(int(rng["bip"][(inst * 31 + i * 7 + j) % 2000] % (1 << q)))
                j += 1
        hot = [sorted(h) for h in hot]
        brute = set()
        for tup in itertools.product(*hot):
            brute.update(int(a) for a in ora.invert(q, r, delta, seed, np.array(tup, np.uint32)))
        res = ora.reconstruct(q, r, delta, seed, hot)
        assert not res["overflow"]
        assert list(res["addresses"]) == sorted(brute)


def test_oracle_matches_reference_random(ora, ref):
    """Random sliding schedules at the small geometry: identical u16 state,
    hot lists and estimates (bit-exact) between restatement and reference."""
    rng = np.random.default_rng(1)
    for trial in range(6):
        p = abi.small_params(int(rng.integers(1, 1000)))
        a, b = ora.sketch(p), ref.sketch(p)
        for step in range(int(rng.integers(3, 9))):
            pairs = np.zeros(int(rng.integers(0, 3000)), dtype=abi.PAIR_DTYPE)
            pairs["aip"] = 0x0A000000 + rng.integers(0, 40, len(pairs))
            pairs["bip"] = rng.integers(0, 2**32, len(pairs), dtype=np.uint64)
            a.update(pairs)
            b.update(pairs)
            op = rng.integers(0, 3)
            if op == 0:
                a.slide(); b.slide()
            elif op == 1:
                a.reinit(); b.reinit()
        for x, y in zip(a.cells(), b.cells()):
            assert np.array_equal(x, y)
        for k in (1, 2, 3, 7):
            ha, hb = a.extract_hot(k, 5), b.extract_hot(k, 5)
            assert all(np.array_equal(x, y) for x, y in zip(ha, hb))
            fa, sa = a.estimate_context(k, 3)
            fb, sb = b.estimate_context(k, 3)
            assert np.array_equal(fa, fb) and sa == sb
            for aip in range(0x0A000000, 0x0A000000 + 40, 7):
                ea, eb = a.estimate(aip, k), b.estimate(aip, k)
                assert (ea.value, ea.usle_weight, ea.saturated) == (eb.value, eb.usle_weight,
                                                                   eb.saturated)


def test_oracle_errors(ora):
    with pytest.raises(abi.ConfigError):
        ora.validate(abi.Params(delta=3))  # (r-2)*delta + q < 32
    with pytest.raises(abi.ConfigError):
        ora.validate(abi.Params(eta_prime=1))
    p = abi.small_params(1)
    wc = abi.WindowConfig(k=0)
    with pytest.raises(abi.ConfigError):
        ora.engine(p, wc)
    e = ora.engine(p, abi.WindowConfig(k=2, theta=64))
    rec = np.zeros(2, dtype=abi.RECORD_DTYPE)
    rec["ts_us"] = [5_000_000, 3_000_000]
    with pytest.raises(abi.OrderingError):
        e.process(rec)
    a, b = ora.sketch(p), ora.sketch(p)
    b.slide()
    with pytest.raises(abi.IncompatibleSketchError):
        a.merge_min(b)
