"""Incremental window tracking of persistent engine batches (detect.cu
phase_a_inc, srlg_internal.cuh IncDev) against the full per-detection sweep
and the CPU oracle. Every detection of a launch after the first re-examines
only the state blocks the window moved past or a scan marked (mode 1: RSRA,
mode 2: RSRA and SLEA); reports and final state must be byte-identical in
every mode, to the full sweep (mode 0) and to the oracle
(run_detection, src/window.cpp:36-78) on traces with little churn (Zipf, the
bench's C2 shape), heavy churn (uniform hosts: many cells enter and leave
every slide), short windows, empty slices and raw-packet ingest."""
import numpy as np
import pytest

from paper_1805_09246_b200 import abi, native, synth

pytestmark = pytest.mark.gpu


def _run(params, wc, pairs, off, mode, anet=None):
    e = native.WindowEngine.from_params(params, wc, device=0)
    e.set_incremental(mode)
    if anet is not None:
        e.set_anet(anet)
    e.process_slices(pairs, off)
    e.finish()
    return e, e.take_reports()


def _check(ora, params, wc, pairs, off):
    o = ora.engine(params, wc)
    o.process_slices(pairs, off)
    o.finish()
    expected = o.take_reports()
    runs = {mode: _run(params, wc, pairs, off, mode) for mode in (2, 1, 3, 0)}
    for mode, (e, got) in runs.items():
        assert got == expected, f"incremental mode {mode} differs from the oracle"
    e = runs[2][0]
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    for mode, (e, _) in runs.items():
        assert np.array_equal(e.rsra().cells(), ors), mode
        assert np.array_equal(e.slea().cells(), ole), mode
    return abi.parse_blobs(expected)


@pytest.mark.parametrize("k,slices,packets", [(20, 60, 6_000_000), (3, 40, 2_000_000),
                                              (1, 12, 600_000)])
def test_zipf_low_churn(ora, k, slices, packets):
    w = synth.scaled(synth.WORKLOADS["c2"], packets=packets, n_slices=slices, planted=40,
                     planted_spread=max(1, k))
    pairs, off = synth.trace(w).generate()
    reps = _check(ora, w.sketch_params(), w.window_config(k=k, t0_us=0), pairs, off)
    assert len(reps) >= slices - k + 1
    assert sum(len(r.entries) for r in reps) > 0


@pytest.mark.parametrize("k", [2, 7])
def test_uniform_high_churn(ora, k):
    """uniform background hosts: most cells of a slice are new, and as many
    leave the window every slide (every block of the state is re-examined
    again and again)"""
    w = synth.scaled(synth.WORKLOADS["c5"], packets=4_000_000, n_slices=30, ddos_sources=400_000)
    pairs, off = synth.trace(w).generate()
    reps = _check(ora, w.sketch_params(), w.window_config(k=k, t0_us=0), pairs, off)
    assert any(r.entries for r in reps)


def test_empty_slices_and_bursts(ora):
    """slices without records between busy ones: the window moves past whole
    slices nobody wrote (exits without any scan in between)"""
    w = synth.scaled(synth.WORKLOADS["c2"], packets=3_000_000, n_slices=24, planted=20,
                     planted_spread=4)
    pairs, off = synth.trace(w).generate()
    # drop the records of slices 6..9 and 15: their offsets collapse
    keep = np.ones(len(pairs), dtype=bool)
    for s in (6, 7, 8, 9, 15):
        keep[off[s]:off[s + 1]] = False
    sizes = np.diff(off)
    for s in (6, 7, 8, 9, 15):
        sizes[s] = 0
    off2 = np.concatenate([[0], np.cumsum(sizes)]).astype(off.dtype)
    _check(ora, w.sketch_params(), w.window_config(k=5, t0_us=0), pairs[keep], off2)


def test_small_geometry(ora):
    """the reference's small geometry (tests/test_window.cpp:16-30): few
    blocks (CTA ranges of a block or two, the last SLEA block partial) and
    SLEA rows of 2296 cells, so blocks straddle rows"""
    p = abi.small_params(5)
    rng = np.random.default_rng(3)
    n_sl, per = 30, 20_000
    pairs = np.zeros(n_sl * per, dtype=abi.PAIR_DTYPE)
    # 40 busy hosts whose peers turn over (new peers every slice, old ones
    # leave the window), over a fixed set of quiet background pairs
    pairs["aip"] = 0x0A000000 + rng.integers(0, 40, len(pairs))
    pairs["bip"] = rng.integers(0, 2**32, len(pairs), dtype=np.uint64)
    quiet = rng.integers(0, 2, len(pairs)).astype(bool)
    pairs["aip"][quiet] = 0x0B000000 + rng.integers(0, 5000, quiet.sum())
    pairs["bip"][quiet] = 0x0C000000 + rng.integers(0, 3, quiet.sum())
    off = np.arange(0, n_sl * per + 1, per, dtype=np.uint64)
    wc = abi.WindowConfig(k=4, slice_us=1000, theta=64, t0_us=0)
    _check(ora, p, wc, pairs, off)


def test_raw_packet_ingest_tracked():
    """raw packets classified inside the tracked scan (trace.cpp:111-116)"""
    w = synth.scaled(synth.WORKLOADS["c2"], packets=2_000_000, n_slices=16, planted=20,
                     planted_spread=3)
    pairs, off = synth.trace(w).generate()
    anet = abi.Anet.of(["10.0.0.0/8", "192.168.1.0/24"])
    params, wc = w.sketch_params(), w.window_config(k=3, t0_us=0)
    got = []
    for mode in (2, 1, 0):
        e, reps = _run(params, wc, pairs, off, mode, anet=anet)
        got.append((reps, e.rsra().cells(), e.slea().cells()))
    for g in got[:2]:
        assert g[0] == got[2][0]
        assert np.array_equal(g[1], got[2][1]) and np.array_equal(g[2], got[2][2])


def test_mode_argument():
    e = native.WindowEngine.from_params(abi.small_params(1), abi.WindowConfig(k=3), device=0)
    with pytest.raises(abi.InvalidArgument):
        e.set_incremental(4)


@pytest.mark.parametrize("ctas,groups", [(16, 1), (24, 3), (16, 4), (40, 8), (9, 2)])
def test_reconstruction_groups(ora, ctas, groups):
    """the reconstruction pipeline with 1..8 groups (groups + 1 buffer sets in
    flight; detection d on group d % groups, set d % (groups + 1)): reports
    and state identical to the oracle"""
    w = synth.scaled(synth.WORKLOADS["c2"], packets=4_000_000, n_slices=40, planted=40,
                     planted_spread=6)
    pairs, off = synth.trace(w).generate()
    params, wc = w.sketch_params(), w.window_config(k=6, t0_us=0)
    o = ora.engine(params, wc)
    o.process_slices(pairs, off)
    o.finish()
    e = native.WindowEngine.from_params(params, wc, device=0)
    e.set_recon(ctas, groups)
    e.process_slices(pairs, off)
    e.finish()
    assert e.take_reports() == o.take_reports()
    ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), ors) and np.array_equal(e.slea().cells(), ole)
    with pytest.raises(abi.InvalidArgument):
        e.set_recon(16, 9)


def test_successive_launches(ora):
    """several process_slices calls on one engine (one launch each): every
    launch's init detection rebuilds the tracking structures from the state
    the previous launch left"""
    w = synth.scaled(synth.WORKLOADS["c2"], packets=5_000_000, n_slices=50, planted=30,
                     planted_spread=5)
    pairs, off = synth.trace(w).generate()
    params, wc = w.sketch_params(), w.window_config(k=8, t0_us=0)
    o = ora.engine(params, wc)
    o.process_slices(pairs, off)
    o.finish()
    expected = o.take_reports()
    for mode in (1, 0):
        e = native.WindowEngine.from_params(params, wc, device=0)
        e.set_incremental(mode)
        cuts = [0, 9, 10, 27, 50]
        for a, b in zip(cuts[:-1], cuts[1:]):
            sub = off[a:b + 1]
            e.process_slices(pairs[int(sub[0]):int(sub[-1])], sub - sub[0], first_slice=a)
        e.finish()
        assert e.take_reports() == expected, mode
        ors, ole = o.cells(e.rsra().num_cells, e.slea().num_cells)
        assert np.array_equal(e.rsra().cells(), ors) and np.array_equal(e.slea().cells(), ole)
