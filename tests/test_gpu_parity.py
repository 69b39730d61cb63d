"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference-generated golden fixtures. Integer state must be bit-exact (u16
distances exported from the u32 stamps); reports byte-identical, which makes
estimates bit-identical (tolerance 0, well inside north_star's 1e-6)."""
import json

import numpy as np
import pytest

from paper_1805_09246_b200 import abi, native, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden(golden_dir):
    return dict(states=np.load(golden_dir / "states.npz"),
                reports=np.load(golden_dir / "reports.npz"),
                rec=json.loads((golden_dir / "reconstruct.json").read_text()))


def gpu_pair(params, device=0):
    return (native.Rsra(native.rsra_config(params), device),
            native.Slea(native.slea_config(params), device))


def rand_pairs(rng, n, hosts=40):
    p = np.zeros(n, dtype=abi.PAIR_DTYPE)
    p["aip"] = 0x0A000000 + rng.integers(0, hosts, n)
    p["bip"] = rng.integers(0, 2**32, n, dtype=np.uint64)
    return p


def assert_same_state(rs, le, sk):
    ors, ole = sk.cells()
    assert np.array_equal(rs.cells(), ors)
    assert np.array_equal(le.cells(), ole)


@pytest.mark.parametrize("params", [abi.small_params(3), abi.Params(seed=808)],
                         ids=["small", "default"])
def test_scan_state_bitexact_vs_oracle(ora, params):
    rng = np.random.default_rng(7)
    rs, le = gpu_pair(params)
    sk = ora.sketch(params)
    for step in range(8):
        pairs = rand_pairs(rng, int(rng.integers(0, 50_000)))
        native.update_pairs(rs, le, pairs)
        sk.update(pairs)
        assert_same_state(rs, le, sk)
        op = step % 3
        if op == 0:
            rs.slide(); le.slide(); sk.slide()
        elif op == 1:
            rs.reinitialize(); le.reinitialize(); sk.reinit()
        assert rs.slides == sk.slides
    assert_same_state(rs, le, sk)


@pytest.mark.parametrize("name,params", [("small_seed7", abi.small_params(7)),
                                         ("small_seed9_reinit", abi.small_params(9)),
                                         ("default_seed1", abi.Params())])
def test_golden_states(ora, golden, name, params):
    st = golden["states"]
    rs, le = gpu_pair(params)
    sched = st[f"{name}__schedule"]
    pool = ora.rng_pair_array(42, int(sched[:, 0].sum()))
    off = 0
    for n, op in sched:
        native.update_pairs(rs, le, pool[off: off + int(n)])
        off += int(n)
        if op == 1:
            rs.slide(); le.slide()
        elif op == 2:
            rs.reinitialize(); le.reinitialize()
    assert np.array_equal(rs.cells(), st[f"{name}__rsra"])
    assert np.array_equal(le.cells(), st[f"{name}__slea"])


def test_saturation_across_65535_slides(ora):
    """One cell set, then 70,000 slides: distances saturate at 0xFFFF exactly
    like counter_ops::slide (sliding_counters.cpp:18-22)."""
    # tiny geometry so the O(cells) oracle slide stays cheap
    p = abi.Params(q=12, r=5, delta=7, eta=1, q_prime=2, r_prime=1, delta_prime=2, eta_prime=4,
                   theta=64, seed=2)
    rs, le = gpu_pair(p)
    sk = ora.sketch(p)
    pairs = rand_pairs(np.random.default_rng(3), 64)
    native.update_pairs(rs, le, pairs)
    sk.update(pairs)
    for target in (1, 65533, 65534, 65535, 65536, 70000):
        while rs.slides < target:
            rs.slide(); le.slide(); sk.slide()
        assert_same_state(rs, le, sk)
        ref_w = sk.estimate_context(65534, 1)[0]
        assert np.array_equal(le.estimate_context(65534)[0], ref_w)
        assert (ref_w[0] > 0) == (target < 65534)


@pytest.mark.parametrize("k", [1, 2, 3, 7, 300, 65534])
def test_window_queries_vs_oracle(ora, k):
    p = abi.Params(seed=5)
    rs, le = gpu_pair(p)
    sk = ora.sketch(p)
    w = synth.scaled(synth.WORKLOADS["c2"], packets=400_000, n_slices=8, planted=20,
                     planted_spread=4)
    pairs, off = synth.trace(w).generate()
    for s in range(8):
        chunk = pairs[off[s]: off[s + 1]]
        native.update_pairs(rs, le, chunk)
        sk.update(chunk)
        if s < 7:
            rs.slide(); le.slide(); sk.slide()
    hg = rs.extract_hot(k)
    ho = sk.extract_hot(k, 5)
    assert all(np.array_equal(a, b) for a, b in zip(hg, ho))
    fg, sfg = le.estimate_context(k)
    fo, sfo = sk.estimate_context(k, 5)
    assert np.array_equal(fg, fo) and sfg == sfo
    aips = np.concatenate([np.array([a for a, _ in synth.trace(w).planted()], np.uint32),
                           np.arange(0x0A000001, 0x0A000001 + 300, dtype=np.uint32)])
    wg = le.usle_weights(k, aips)
    for aip, wgt in zip(aips[::7], wg[::7]):
        e = sk.estimate(int(aip), k)
        assert e.usle_weight == wgt
        g = le.estimate(int(aip), k, sfg)
        assert (g.value, g.corrected_weight, g.saturated) == (e.value, e.corrected_weight,
                                                              e.saturated)


def test_reconstruct_golden(golden):
    for c in golden["rec"]:
        cfg = abi.RsraConfig(q=c["q"], r=c["r"], delta=c["delta"], eta=8, tau=3,
                             seed_rhfg0=c["seed"])
        if (c["r"] - 2) * c["delta"] + c["q"] < 32:
            # the reference builds these groups standalone (no Rsra): use a
            # covering geometry with the same hash group for q=10 cases is
            # impossible, so compare only covering cases here
            continue
        rs = native.Rsra(cfg)
        res = native.reconstruct(rs, c["hot"])
        assert list(res["addresses"]) == c["addresses"]
        assert res["overflow"] == c["overflow"]
        assert res["tuples_checked"] == c["checked"] and res["tuples_kept"] == c["kept"]
        assert native.reconstruct(rs, c["hot"], tuple_cap=2)["overflow"] == c["overflow_cap2"]


def test_reconstruct_vs_oracle_random(ora):
    rng = np.random.default_rng(11)
    cfg = abi.RsraConfig(q=14, r=5, delta=6, eta=8, tau=3, seed_rhfg0=99)
    rs = native.Rsra(cfg)
    for inst in range(25):
        hot = [set() for _ in range(5)]
        for _ in range(int(rng.integers(0, 6))):
            cols = rs.forward(int(rng.integers(0, 2**32)))
            for i in range(5):
                hot[i].add(int(cols[i]))
        for i in range(5):
            while len(hot[i]) < int(rng.integers(1, 60)):
                hot[i].add(int(rng.integers(0, 1 << 14)))
        hot = [sorted(h) for h in hot]
        for cap in (1 << 22, 50):
            g = native.reconstruct(rs, hot, tuple_cap=cap)
            o = ora.reconstruct(14, 5, 6, 99, hot, tuple_cap=cap)
            assert list(g["addresses"]) == list(o["addresses"])
            assert (g["overflow"], g["tuples_checked"], g["tuples_kept"]) == (
                o["overflow"], o["tuples_checked"], o["tuples_kept"])
    # work cap
    hot = [list(range(0, 3000, 3))] * 5
    g = native.reconstruct(rs, hot, work_cap=10**6)
    assert g["overflow"] and len(g["addresses"]) == 0


@pytest.mark.parametrize("k", [1, 5, 300])
def test_detect_blob_vs_oracle(ora, k):
    p = abi.Params(seed=808)
    rs, le = gpu_pair(p)
    sk = ora.sketch(p)
    w = synth.scaled(synth.WORKLOADS["c2"], packets=600_000, n_slices=6, planted=40,
                     planted_spread=3)
    pairs, off = synth.trace(w).generate()
    for s in range(6):
        chunk = pairs[off[s]: off[s + 1]]
        native.update_pairs(rs, le, chunk)
        sk.update(chunk)
        if s < 5:
            rs.slide(); le.slide(); sk.slide()
    for keep in (0, 1):
        wc = abi.WindowConfig(k=k, theta=1024, keep_below_threshold=keep)
        g = native.run_detection(rs, le, wc, 5, False)
        o = sk.detect(wc, 5, False)
        assert g == o
    reps = abi.parse_blobs(g)
    assert reps[0].candidate_count > 0


def _engine_gpu(params, wcfg):
    return native.WindowEngine.from_params(params, wcfg)


@pytest.mark.parametrize("key,k", [("trace0_k1", 1), ("trace1_k3", 3), ("trace2_k10", 10),
                                   ("trace3_k3", 3)])
@pytest.mark.parametrize("seed", [7, 11])
def test_engine_records_golden(golden, key, k, seed):
    rec = golden["reports"][f"records__{key}"].view(abi.RECORD_DTYPE)
    wc = abi.WindowConfig(k=k, theta=64, t0_us=1_000_000, reinit_per_window=int(k == 1))
    e = _engine_gpu(abi.small_params(seed), wc)
    e.process(rec)
    e.finish()
    assert e.take_reports() == golden["reports"][f"engine__{key}__seed{seed}"].tobytes()


def test_engine_full_geometry_golden(golden):
    rep = golden["reports"]
    w = synth.scaled(synth.WORKLOADS["c1"], packets=1 << 18, planted=20, bg_hosts=100_000)
    pairs, off = synth.trace(w).generate()
    e = _engine_gpu(w.sketch_params(), w.window_config(t0_us=0))
    e.process_slices(pairs, off)
    e.finish()
    assert e.take_reports() == rep["c1small__engine"].tobytes()
    w2 = synth.scaled(synth.WORKLOADS["c2"], packets=1_200_000, n_slices=12, planted_spread=5,
                      planted=30)
    pairs2, off2 = synth.trace(w2).generate()
    e = _engine_gpu(w2.sketch_params(), w2.window_config(k=5, t0_us=0))
    e.process_slices(pairs2, off2)
    e.finish()
    assert e.take_reports() == rep["c2small__engine"].tobytes()


def test_engine_device_input_and_state(ora):
    """Pairs resident in HBM (the benchmark path) give the same reports and the
    same final state as host input and as the oracle engine."""
    import torch

    w = synth.scaled(synth.WORKLOADS["c2"], packets=2_000_000, n_slices=20, planted=30,
                     planted_spread=10)
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(k=10, t0_us=0)
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    ref_blob = o.take_reports()
    d = torch.from_numpy(pairs.view(np.uint8)).cuda()
    torch.cuda.synchronize()
    e = _engine_gpu(w.sketch_params(), wc)
    e.process_slices(offsets=off, device_ptr=d.data_ptr())
    e.finish()
    assert e.take_reports() == ref_blob
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), ors)
    assert np.array_equal(e.slea().cells(), ole)
    # reset + replay through the host path
    e.reset()
    e.process_slices(pairs, off)
    e.finish()
    assert e.take_reports() == ref_blob


@pytest.mark.parametrize("policy", [0, 1, 2])
def test_partition_merge_bitexact(ora, golden, policy):
    """acceptance [2]: 4 partitions merged (distance min == stamp max) are
    bit-exact with the whole, on the device."""
    p = abi.Params(seed=9)
    w = synth.scaled(synth.WORKLOADS["c2"], packets=900_000, n_slices=3, planted=10,
                     planted_spread=3)
    pairs, off = synth.trace(w).generate()
    parts = [gpu_pair(p) for _ in range(4)]
    whole = gpu_pair(p)
    for s in range(3):
        chunk = pairs[off[s]: off[s + 1]]
        if policy == 0:  # any partition is exact; a random one here
            route = np.random.default_rng(s).integers(0, 4, len(chunk))
        elif policy == 1:
            route = np.arange(len(chunk)) % 4
        else:
            route = (chunk["aip"] >> 24) % 4
        for n in range(4):
            native.update_pairs(*parts[n], chunk[route == n])
        native.update_pairs(*whole, chunk)
        for x in parts + [whole]:
            x[0].slide(); x[1].slide()
    mr, ml = parts[0]
    for n in range(1, 4):
        mr.merge_min(parts[n][0])
        ml.merge_min(parts[n][1])
    assert np.array_equal(mr.cells(), whole[0].cells())
    assert np.array_equal(ml.cells(), whole[1].cells())
    sk = ora.sketch(p)
    for s in range(3):
        sk.update(pairs[off[s]: off[s + 1]])
        sk.slide()
    assert_same_state(mr, ml, sk)


def test_merge_incompatible_and_import_export(ora):
    p = abi.small_params(4)
    a, al = gpu_pair(p)
    b, bl = gpu_pair(p)
    b.slide()
    assert a.compatibility_mismatch(b) == "slice position"
    with pytest.raises(abi.IncompatibleSketchError):
        a.merge_min(b)
    # cells_mut-style write-back then read (test_slea.cpp:95-116 toy row)
    tiny = abi.SleaConfig(q=1, r=1, delta=2, eta=6, seed_h3=1)
    tiny.seeds_lh[0] = 2
    t = native.Slea(tiny)
    assert t.row_length == 8
    t.set_cells(np.array([0, 1, 2, 3, 0xFFFF, 0xFFFF, 0xFFFF, 0xFFFF], np.uint16))
    f, _ = t.estimate_context(3)
    assert f[0] == 3.0 / 8.0
    t.set_cells(np.zeros(8, np.uint16))
    assert t.estimate_context(1)[0][0] == 1.0
    assert np.array_equal(t.cells(), np.zeros(8, np.uint16))
    with pytest.raises(abi.SaturationError):
        t.estimate(0x0A000001, 1)
    # import/export round trip with arbitrary distances, then slide + merge
    rng = np.random.default_rng(5)
    cells = rng.integers(0, 70000, a.num_cells).clip(0, 0xFFFF).astype(np.uint16)
    a.set_cells(cells)
    assert np.array_equal(a.cells(), cells)
    a.set_slides(17)
    assert np.array_equal(a.cells(), cells)
    sk = ora.sketch(p)
    sk.set_cells(cells, None)
    a.slide(); sk.slide()
    assert np.array_equal(a.cells(), sk.cells()[0])


def test_clone_is_deep():
    p = abi.small_params(4)
    a, al = gpu_pair(p)
    native.update_pairs(a, al, rand_pairs(np.random.default_rng(1), 5000))
    b = a.clone()
    bl = al.clone()
    native.update_pairs(a, al, rand_pairs(np.random.default_rng(2), 5000))
    assert not np.array_equal(a.cells(), b.cells())
    c = b.clone()
    assert np.array_equal(c.cells(), b.cells())
    assert np.array_equal(bl.clone().cells(), bl.cells())


@pytest.mark.parametrize("checker", ["ora", "ref"])
def test_c1_full_size_vs_oracle(request, checker):
    """C1 at full size (2^20 packets, one discrete slice, paper geometry):
    state bit-exact and identical report, against the C restatement and
    against the reference library itself (oracle/_ref)."""
    be = request.getfixturevalue(checker)
    w = synth.WORKLOADS["c1"]
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(t0_us=0)
    o = be.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    e = _engine_gpu(w.sketch_params(), wc)
    e.process_slices(pairs, off)
    e.finish()
    assert e.take_reports() == o.take_reports()
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), ors)
    assert np.array_equal(e.slea().cells(), ole)


@pytest.mark.slow
def test_c2_full_size_reports_vs_oracle(ora):
    """C2 at full size (100M packets, 600 slices, k=300): all 301 reports
    byte-identical with the oracle engine, final state bit-exact."""
    w = synth.WORKLOADS["c2"]
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(t0_us=0)
    e = _engine_gpu(w.sketch_params(), wc)
    e.process_slices(pairs, off)
    e.finish()
    got = e.take_reports()
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    exp = o.take_reports()
    assert len(abi.parse_blobs(got)) == 301
    assert got == exp
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), ors)
    assert np.array_equal(e.slea().cells(), ole)


@pytest.mark.slow
def test_c5_ddos_full_size_vs_oracle(ora):
    """C5 at full size (100M packets, one victim with 10M distinct sources over
    uniform background): every report identical with the oracle; the victim
    is detected with a saturated SLEA estimate (eta' ln eta'), no background
    host is ever reported."""
    w = synth.WORKLOADS["c5"]
    tr = synth.trace(w)
    pairs, off = tr.generate()
    wc = w.window_config(t0_us=0)
    e = _engine_gpu(w.sketch_params(), wc)
    e.process_slices(pairs, off)
    e.finish()
    got = e.take_reports()
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    assert got == o.take_reports()
    victim = tr.victim_aip()
    reps = abi.parse_blobs(got)
    assert len(reps) == 301
    hosts = {aip for r in reps for aip, _, _ in r.entries}
    assert hosts == {victim}
    sat = [est for r in reps for aip, est, s in r.entries if s]
    assert sat and all(abs(v - 16384 * np.log(16384)) < 1e-6 for v in sat)


@pytest.mark.slow
def test_c4_geometry_exceeding_l2_vs_oracle(ora):
    """C4's geometry (q'=21: 167.8M SLEA cells, 671 MB of stamps, larger than
    L2) on a 20M-packet, 120-slice trace with k=60: reports and state
    identical with the oracle."""
    w = synth.scaled(synth.WORKLOADS["c4"], packets=20_000_000, n_slices=120,
                     planted_spread=60)
    w = synth.Workload(w.name, w.spec, w.params, 60, False)
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(t0_us=0)
    e = _engine_gpu(w.sketch_params(), wc)
    e.process_slices(pairs, off)
    e.finish()
    got = e.take_reports()
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    assert got == o.take_reports()
    assert len(abi.parse_blobs(got)) == 61
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), ors)
    assert np.array_equal(e.slea().cells(), ole)


def test_c4_geometry_dynamic_scan_chunks_vs_oracle(ora):
    """C4's geometry with slices of ~1.3M pairs (>= 8192 per stream CTA): the
    scans claim their chunks dynamically (detect.cu scan_dynamic) while the
    SLEA is tracked and reconstructed by one group; device and pinned host
    input. Reports and state identical with the oracle."""
    import torch

    w = synth.scaled(synth.WORKLOADS["c4"], packets=5_200_000, n_slices=4, planted=30,
                     planted_spread=2)
    w = synth.Workload(w.name, w.spec, w.params, 2, False)
    pairs, off = synth.trace(w).generate()
    assert np.diff(off).min() >= 8192 * 148
    wc = w.window_config(t0_us=0)
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    expected = o.take_reports()
    assert len(abi.parse_blobs(expected)) == 3
    d = torch.from_numpy(pairs.view(np.uint8)).cuda()
    pinned = torch.from_numpy(pairs.view(np.uint8)).pin_memory()
    torch.cuda.synchronize()
    ors = ole = None
    for mode in ("device", "host_pinned"):
        e = _engine_gpu(w.sketch_params(), wc)
        if mode == "device":
            e.process_slices(offsets=off, device_ptr=d.data_ptr())
        else:
            e.process_slices_host_ptr(pinned.data_ptr(), off)
        e.finish()
        assert e.take_reports() == expected, mode
        if ors is None:
            ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
        assert np.array_equal(e.rsra().cells(), ors), mode
        assert np.array_equal(e.slea().cells(), ole), mode


@pytest.mark.slow
def test_c4_bench_geometry_vs_reference(ref):
    """C4 exactly as bench.py runs it (10^9 packets, 600 slices of 1.67M,
    q'=21: 692 MB of state, k=300, 301 reports) against the reference
    library's own WindowEngine with every host thread: all reports
    byte-identical, final state bit-exact."""
    import os

    import torch

    w = synth.WORKLOADS["c4"]
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(t0_us=0, workers=os.cpu_count() or 1)
    e = _engine_gpu(w.sketch_params(), wc)
    d = torch.from_numpy(pairs.view(np.uint8)).cuda()
    torch.cuda.synchronize()
    e.process_slices(offsets=off, device_ptr=d.data_ptr())
    e.finish()
    got = e.take_reports()
    del d
    o = ref.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    assert len(abi.parse_blobs(got)) == 301
    assert got == o.take_reports()
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), ors)
    assert np.array_equal(e.slea().cells(), ole)


def test_permutation_invariance_full_slice():
    """Order of packets within a slice cannot matter (test_rsra.cpp:88-102)."""
    w = synth.scaled(synth.WORKLOADS["c2"], packets=5_000_000, n_slices=1, planted=50,
                     planted_spread=1)
    pairs, off = synth.trace(w).generate()
    p = w.sketch_params()
    a = gpu_pair(p)
    b = gpu_pair(p)
    native.update_pairs(*a, pairs)
    native.update_pairs(*b, pairs[np.random.default_rng(0).permutation(len(pairs))])
    assert np.array_equal(a[0].stamps()[0], b[0].stamps()[0])
    assert np.array_equal(a[1].stamps()[0], b[1].stamps()[0])


@pytest.mark.parametrize("planted,k", [(300, 1), (700, 1)])
def test_detect_grid_wide_reconstruction_vs_oracle(ora, planted, k):
    """Hot lists large enough that the fused detection kernel reconstructs
    with the whole grid (seed work > 2^21 checks) instead of inside one CTA;
    reports must still equal the oracle's, overflow decisions included."""
    w = synth.scaled(synth.WORKLOADS["c2"], packets=3_000_000, n_slices=1, planted=planted,
                     planted_spread=1, planted_min=1500, planted_max=3000)
    pairs, off = synth.trace(w).generate()
    p = w.sketch_params()
    rs, le = gpu_pair(p)
    sk = ora.sketch(p)
    native.update_pairs(rs, le, pairs)
    sk.update(pairs)
    for cap in (1 << 22, 5000):
        wc = abi.WindowConfig(k=k, theta=1024, tuple_cap=cap)
        g = native.run_detection(rs, le, wc, 0, True)
        o = sk.detect(wc, 0, True)
        assert g == o
    rep = abi.parse_blobs(g)[0]
    assert min(rep.hot_per_row) ** 3 > (1 << 21)


@pytest.mark.parametrize("k,reinit,slices,packets", [(1, 1, 12, 600_000), (4, 0, 30, 3_000_000),
                                                     (25, 0, 40, 12_000_000),
                                                     (2, 0, 7, 9_000_000)])
def test_engine_persistent_batches_vs_per_slice_and_oracle(ora, k, reinit, slices, packets):
    """Persistent batches (one cooperative launch per run of slices, windows
    finalised from the mapped ring while the kernel runs) against per-slice
    launches and the oracle: identical reports and state, for device input
    and for host input split into staging chunks (pageable and pinned; the
    last case has slices spanning several 1 M-pair chunks, which arrive over
    two copy streams)."""
    import torch

    w = synth.scaled(synth.WORKLOADS["c2"], packets=packets, n_slices=slices, planted=40,
                     planted_spread=max(1, k))
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(k=k, t0_us=0, reinit_per_window=reinit)
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    expected = o.take_reports()
    ors, ole = o.cells(0, 0) if False else (None, None)
    d = torch.from_numpy(pairs.view(np.uint8)).cuda()
    torch.cuda.synchronize()
    outs = []
    pinned = torch.from_numpy(pairs.view(np.uint8)).pin_memory()
    for mode in ("device", "host", "per_slice", "host_pinned"):
        e = _engine_gpu(w.sketch_params(), wc)
        if mode == "per_slice":
            e.set_persistent(False)
        if mode == "device":
            e.process_slices(offsets=off, device_ptr=d.data_ptr())
        elif mode == "host_pinned":
            e.process_slices_host_ptr(pinned.data_ptr(), off)
        else:
            e.process_slices(pairs, off)
        e.finish()
        outs.append(e.take_reports())
        if ors is None:
            ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
        assert np.array_equal(e.rsra().cells(), ors), mode
        assert np.array_equal(e.slea().cells(), ole), mode
        if mode == "device":
            us, nwin = e.detect_latency()
            assert nwin == max(0, slices - k) and (nwin == 0 or us > 0)
    assert all(out == expected for out in outs)


@pytest.mark.parametrize("k,reinit", [(10, 0), (1, 1)])
def test_engine_distributed_mode_single_rank_vs_oracle(ora, k, reinit):
    """The multi-GPU path (touched-cell marks -> NCCL max-reduce -> root
    applies stamps -> detection) run with a 1-rank NCCL communicator: the
    root's reports and final state equal the oracle engine's."""
    import torch

    w = synth.scaled(synth.WORKLOADS["c2"], packets=1_500_000, n_slices=15, planted=25,
                     planted_spread=5)
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(k=k, t0_us=0, reinit_per_window=reinit)
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    expected = o.take_reports()
    comm = native.nccl_comm_create(1, native.nccl_unique_id(), 0, 0)
    try:
        e = _engine_gpu(w.sketch_params(), wc)
        e.set_merge(comm, 0, 1, 0)
        d = torch.from_numpy(pairs.view(np.uint8)).cuda()
        torch.cuda.synchronize()
        e.process_slices(offsets=off, device_ptr=d.data_ptr())
        e.finish()
        assert e.take_reports() == expected
        ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
        assert np.array_equal(e.rsra().cells(), ors)
        assert np.array_equal(e.slea().cells(), ole)
        st = e.merge_stats()
        assert st["slice_merges"] == 15
        assert st["bytes_exchanged"] == 15 * (e.rsra().num_cells + e.slea().num_cells)
        del e
    finally:
        native.nccl_comm_destroy(comm)


@pytest.mark.parametrize("arena", [0, 1024])
def test_engine_candidate_tails_over_many_windows(ref, arena):
    """Windows with more candidates than the 1024 the engine writes straight
    to the host, over many windows of one persistent batch: the rest go
    through a ring the host frees as it drains the reports (a 1024-candidate
    ring makes the kernel wait for the host several times). Reports equal the
    reference's own engine's (reconstruct.cpp:32-151; its work_cap of 2^32
    brute-force checks bounds a window at ~1600 candidates)."""
    import os

    import torch

    w = synth.scaled(synth.WORKLOADS["c2"], packets=1200 * 2500 * 8 // 2, n_slices=8,
                     planted=1200, planted_spread=1, planted_min=1500, planted_max=3000)
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(k=2, t0_us=0, workers=os.cpu_count() or 1)
    o = ref.engine(w.sketch_params(), wc)
    o.process_slices(pairs, off)
    o.finish()
    expected = o.take_reports()
    reps = abi.parse_blobs(expected)
    assert sum(r.candidate_count > 1024 for r in reps) >= 6
    e = native.WindowEngine.from_params(w.sketch_params(), wc)
    e.set_arena(arena)
    d = torch.from_numpy(pairs.view(np.uint8)).cuda()
    torch.cuda.synchronize()
    e.process_slices(offsets=off, device_ptr=d.data_ptr())
    e.finish()
    assert e.take_reports() == expected


def test_process_then_process_slices_in_the_same_slice(ora):
    """records delivered through process() and then the rest of the same
    slice through process_slices(): the slice continues (no ordering error),
    reports and state equal the oracle's record-by-record run"""
    w = synth.scaled(synth.WORKLOADS["c2"], packets=400_000, n_slices=4, planted=10,
                     planted_spread=2)
    pairs, off = synth.trace(w).generate()
    wc = w.window_config(k=2, t0_us=0)
    recs = synth.records(pairs, off, wc.slice_us)
    # slice 1's records carry a timestamp half way into the slice; its first
    # half arrives through process(), the rest pre-sliced (placed at the
    # slice start, which is not a regression within the open slice)
    a, b = int(off[1]), int(off[1] + (off[2] - off[1]) // 2)
    recs["ts_us"][a:int(off[2])] += wc.slice_us // 2
    e = _engine_gpu(w.sketch_params(), wc)
    e.process(recs[:b])
    rest_off = np.array([0, off[2] - b, off[3] - b, off[4] - b], dtype=np.uint64)
    e.process_slices(pairs[b:], rest_off, first_slice=1)
    e.finish()
    o = ora.engine(w.sketch_params(), wc)
    o.process(recs)
    o.finish()
    assert e.take_reports() == o.take_reports()


@pytest.mark.parametrize("r,delta,q", [(6, 5, 12), (7, 4, 12), (8, 4, 12), (10, 3, 12)])
def test_rsra_row_counts_vs_oracle(ora, r, delta, q):
    """RSRA row counts other than the paper's 5: the depth-first growth keeps
    its tuple in registers up to 8 rows and walks with its state in the
    per-thread scratch beyond (detect.cu dfs_pairs / dfs_deep); engine
    reports and state byte-identical to the oracle. (3 and 4 rows constrain
    the reconstruction so little that the CPU oracle needs minutes.)"""
    p = abi.Params(q=q, r=r, delta=delta, eta=8, q_prime=8, r_prime=3, delta_prime=8,
                   eta_prime=256, theta=64, seed=r)
    rng = np.random.default_rng(r)
    n_sl, per = 12, 30_000
    pairs = rand_pairs(rng, n_sl * per, hosts=60)
    off = np.arange(0, n_sl * per + 1, per, dtype=np.uint64)
    wc = abi.WindowConfig(k=3, slice_us=1000, theta=64, t0_us=0)
    o = ora.engine(p, wc)
    o.process_slices(pairs, off)
    o.finish()
    expected = o.take_reports()
    e = _engine_gpu(p, wc)
    e.process_slices(pairs, off)
    e.finish()
    got = e.take_reports()
    assert got == expected
    assert sum(len(x.entries) for x in abi.parse_blobs(got)) > 0
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), ors) and np.array_equal(e.slea().cells(), ole)
