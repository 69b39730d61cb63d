"""Raw-packet ingest: classify (trace.cpp:111-116) fused
into the scan. A raw packet {src, dst} yields one record per endpoint inside
the monitored network (src first). CPU: a numpy restatement against the
reference's own classify; GPU: the fused device path against the reference
classification followed by the plain record path (state and reports
bit-exact, record counts equal)."""
import numpy as np
import pytest

from paper_1805_09246_b200 import abi, synth

ANET = ["10.0.0.0/8", "192.168.1.0/24", "172.16.0.0/12"]


def raw_packets(seed, n):
    """a mix of inbound, outbound, internal and foreign packets"""
    rng = np.random.default_rng(seed)
    inside = lambda k: np.where(rng.random(k) < 0.5,  # noqa: E731
                                0x0A000000 + rng.integers(0, 300, k),
                                0xC0A80100 + rng.integers(0, 256, k)).astype(np.uint64)
    outside = lambda k: rng.integers(0x20000000, 0x60000000, k, dtype=np.uint64)  # noqa: E731
    kind = rng.integers(0, 4, n)
    src = np.where(kind < 2, inside(n), outside(n))
    dst = np.where((kind == 1) | (kind == 2), inside(n), outside(n))
    p = np.zeros(n, dtype=abi.PAIR_DTYPE)
    p["aip"], p["bip"] = src, dst
    return p


def classify_np(raw, prefixes):
    """restatement of classify / CidrPrefix::contains (trace.hpp:38-57)"""
    def contains(ip):
        m = np.zeros(len(ip), dtype=bool)
        for pre in prefixes:
            a, b = pre.split("/")
            o = [int(x) for x in a.split(".")]
            addr, bits = (o[0] << 24) | (o[1] << 16) | (o[2] << 8) | o[3], int(b)
            mask = 0 if bits == 0 else (0xFFFFFFFF << (32 - bits)) & 0xFFFFFFFF
            m |= (ip.astype(np.uint64) & mask) == (addr & mask)
        return m

    s_in, d_in = contains(raw["aip"]), contains(raw["bip"])
    out = []
    for i in range(len(raw)):
        if s_in[i]:
            out.append((raw["aip"][i], raw["bip"][i]))
        if d_in[i]:
            out.append((raw["bip"][i], raw["aip"][i]))
    return np.array(out, dtype=abi.PAIR_DTYPE)


def test_classify_restatement_matches_reference(ref):
    raw = raw_packets(1, 5000)
    got = classify_np(raw, ANET)
    exp = ref.classify(raw, abi.Anet.of(ANET))
    assert np.array_equal(got, exp)


@pytest.mark.gpu
def test_update_raw_vs_reference_classify(ref):
    from paper_1805_09246_b200 import native

    p = abi.small_params(5)
    rs, le = native.Rsra(native.rsra_config(p)), native.Slea(native.slea_config(p))
    rs2, le2 = native.Rsra(native.rsra_config(p)), native.Slea(native.slea_config(p))
    anet = abi.Anet.of(ANET)
    for step in range(4):
        raw = raw_packets(10 + step, 20000)
        recs = ref.classify(raw, anet)
        n = native.update_raw(rs, le, raw, anet)
        native.update_pairs(rs2, le2, recs)
        assert n == len(recs)
        assert np.array_equal(rs.cells(), rs2.cells())
        assert np.array_equal(le.cells(), le2.cells())
        for h in (rs, le, rs2, le2):
            h.slide()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["persistent_device", "persistent_host", "per_slice"])
def test_engine_raw_ingest_vs_reference(ref, ora, mode):
    import torch

    from paper_1805_09246_b200 import native

    w = synth.scaled(synth.WORKLOADS["c2"], packets=600_000, n_slices=16, planted=20,
                     planted_spread=3)
    wc = w.window_config(k=4, t0_us=0)
    anet = abi.Anet.of(ANET)
    slices = [raw_packets(100 + s, 30000) for s in range(16)]
    raw = np.concatenate(slices)
    raw_off = np.cumsum([0] + [len(x) for x in slices]).astype(np.uint64)
    recs = [ref.classify(x, anet) for x in slices]
    rec_all = np.concatenate(recs)
    rec_off = np.cumsum([0] + [len(x) for x in recs]).astype(np.uint64)
    o = ora.engine(w.sketch_params(), wc)
    o.process_slices(rec_all, rec_off)
    o.finish()
    expected = o.take_reports()
    e = native.WindowEngine.from_params(w.sketch_params(), wc)
    e.set_anet(anet)
    if mode == "per_slice":
        e.set_persistent(False)
    if mode == "persistent_device":
        d = torch.from_numpy(raw.view(np.uint8)).cuda()
        e.process_slices(offsets=raw_off, device_ptr=d.data_ptr())
    else:
        e.process_slices(raw, raw_off)
    e.finish()
    assert e.take_reports() == expected
    rs, le = o.cells(e.rsra().num_cells, e.slea().num_cells)
    assert np.array_equal(e.rsra().cells(), rs)
    assert np.array_equal(e.slea().cells(), le)
    assert e.records == len(rec_all)


def timed(packets, slices, t0=1_000_000, slice_us=1_000_000, seed=3):
    """RawPacket / TraceRecord records {ts, a, b} spread over `slices`, time-ordered"""
    rng = np.random.default_rng(seed)
    ts = np.sort(t0 + rng.integers(0, slices * slice_us, len(packets)))
    out = np.zeros(len(packets), dtype=abi.RECORD_DTYPE)
    out["ts_us"], out["aip"], out["bip"] = ts, packets["aip"], packets["bip"]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("raw_mode", [False, True])
def test_engine_binary_trace_file(ref, ora, tmp_path, raw_mode):
    from paper_1805_09246_b200 import native

    p = abi.small_params(9)
    wc = abi.WindowConfig(k=3, theta=64, t0_us=1_000_000)
    anet = abi.Anet.of(ANET)
    pk = raw_packets(55, 60000)
    recs_in = timed(pk, 10)
    path = tmp_path / "trace.bin"
    recs_in.tofile(path)
    if raw_mode:  # the reference classifies each packet, keeping its timestamp
        out = []
        for r in recs_in:
            one = np.zeros(1, dtype=abi.PAIR_DTYPE)
            one["aip"], one["bip"] = r["aip"], r["bip"]
            for c in ref.classify(one, anet):
                out.append((r["ts_us"], c["aip"], c["bip"]))
        expected_recs = np.array(out, dtype=abi.RECORD_DTYPE)
    else:
        expected_recs = recs_in
    o = ora.engine(p, wc)
    o.process(expected_recs)
    o.finish()
    e = native.WindowEngine.from_params(p, wc)
    if raw_mode:
        e.set_anet(anet)
    assert e.process_file(path) == len(recs_in)
    e.finish()
    assert e.take_reports() == o.take_reports()
    assert e.records == len(expected_recs)


@pytest.mark.gpu
def test_engine_binary_trace_file_errors(tmp_path):
    from paper_1805_09246_b200 import native

    e = native.WindowEngine.from_params(abi.small_params(9),
                                        abi.WindowConfig(k=3, theta=64, t0_us=1_000_000))
    with pytest.raises(abi.ParseError, match="cannot open trace file"):
        e.process_file(tmp_path / "missing.bin")
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\0" * 20)
    with pytest.raises(abi.FormatError, match="trailing partial record"):
        e.process_file(bad)
