"""Sketch streams ("SRLG" v1, sketch_io.hpp:13-24 / sketch_io.cpp:106-180).

The fixture tests/golden/sketch_streams.npz holds streams written by the
REFERENCE's own serialize_sketch (tests/golden/make_golden_sketch.py). CPU
tests pin the fixture's layout against the reference's test expectations and
against states.npz (same schedules); GPU tests require the device path to
write byte-identical streams for the same schedule, to read the reference's
streams back into identical state, and to fail like the reference on
malformed input (test_sketch_io.cpp:92-131)."""
import struct

import numpy as np
import pytest

from paper_1805_09246_b200 import abi

CASES = ["small_seed7", "small_seed9_reinit", "default_seed1"]


@pytest.fixture(scope="module")
def streams(golden_dir):
    return np.load(golden_dir / "sketch_streams.npz")


def params_of(streams, name):
    v = [int(x) for x in streams[f"{name}__params"]]
    keys = ("q", "r", "delta", "eta", "q_prime", "r_prime", "delta_prime", "eta_prime", "theta",
            "seed")
    return abi.Params(**dict(zip(keys, v)))


def parse(stream: bytes):
    """independent restatement of the stream layout (sketch_io.cpp:106-134)"""
    assert stream[:4] == b"SRLG"
    version, kind = struct.unpack_from("<HB", stream, 4)
    assert version == 1
    off = 7
    if kind == 1:
        q, r, delta, eta, tau = struct.unpack_from("<5I", stream, off)
        off += 20 + 24
        cfg = dict(q=q, r=r, delta=delta, eta=eta, tau=tau)
    else:
        q, r, delta, eta = struct.unpack_from("<4I", stream, off)
        off += 16 + 8 * (1 + r)
        cfg = dict(q=q, r=r, delta=delta, eta=eta)
    (slides,) = struct.unpack_from("<Q", stream, off)
    off += 8
    return kind, cfg, slides, off, np.frombuffer(stream[off:], dtype="<u2")


# ---------------------------------------------------------------- CPU side

@pytest.mark.parametrize("name", CASES)
def test_fixture_layout(streams, name):
    rs = bytes(streams[f"{name}__rsra"])
    le = bytes(streams[f"{name}__slea"])
    k1, c1, s1, off1, cells1 = parse(rs)
    k2, c2, s2, off2, cells2 = parse(le)
    assert (k1, k2) == (1, 2) and s1 == s2
    assert off1 == 59  # RSRA counters start at byte 59 (test_sketch_io.cpp:121-135)
    assert len(cells1) == (1 << c1["q"]) * c1["r"] * c1["eta"]
    row_len = (1 << c2["q"]) * c2["delta"] + c2["eta"] - c2["delta"]  # slea.hpp:33-35
    assert len(cells2) == row_len * c2["r"]


@pytest.mark.parametrize("name", ["small_seed7", "small_seed9_reinit"])
def test_fixture_matches_states_golden(streams, golden_dir, name):
    """the same schedules as states.npz: identical counters and slides"""
    st = np.load(golden_dir / "states.npz")
    _, _, s1, _, cells1 = parse(bytes(streams[f"{name}__rsra"]))
    _, _, s2, _, cells2 = parse(bytes(streams[f"{name}__slea"]))
    assert np.array_equal(cells1, st[f"{name}__rsra"])
    assert np.array_equal(cells2, st[f"{name}__slea"])
    assert s1 == int(st[f"{name}__slides"][0])


@pytest.mark.parametrize("name", CASES)
def test_reference_reads_fixture(ref, streams, name):
    for which in ("rsra", "slea"):
        data = bytes(streams[f"{name}__{which}"])
        kind, slides, cells = ref.deserialize(data)
        assert kind == (1 if which == "rsra" else 2)
        _, _, s, _, parsed = parse(data)
        assert slides == s and np.array_equal(cells, parsed)


# ---------------------------------------------------------------- GPU side

def gpu_replay(ora, streams, name, native):
    p = params_of(streams, name)
    rs = native.Rsra(native.rsra_config(p))
    le = native.Slea(native.slea_config(p))
    schedule = [tuple(int(x) for x in row) for row in streams[f"{name}__schedule"]]
    pool = ora.rng_pair_array(42, sum(n for n, _ in schedule))
    off = 0
    for n, op in schedule:
        native.update_pairs(rs, le, pool[off: off + n])
        off += n
        if op == 1:
            rs.slide(); le.slide()
        elif op == 2:
            rs.reinitialize(); le.reinitialize()
    return rs, le


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_writes_reference_bytes(ora, streams, name):
    from paper_1805_09246_b200 import native

    rs, le = gpu_replay(ora, streams, name, native)
    assert rs.serialize() == bytes(streams[f"{name}__rsra"])
    assert le.serialize() == bytes(streams[f"{name}__slea"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_reads_reference_streams(streams, name):
    from paper_1805_09246_b200 import native

    for which, cls in (("rsra", native.Rsra), ("slea", native.Slea)):
        data = bytes(streams[f"{name}__{which}"])
        h = native.deserialize_sketch(data)
        assert isinstance(h, cls)
        _, _, slides, _, cells = parse(data)
        assert h.slides == slides
        assert np.array_equal(h.cells(), cells)
        assert h.serialize() == data  # round trip (test_sketch_io.cpp:52-77)


@pytest.mark.gpu
def test_gpu_stream_errors_match_reference(ref, streams):
    from paper_1805_09246_b200 import native

    good = bytes(streams["small_seed7__rsra"])
    bad_cases = {
        "magic": b"SRLX" + good[4:],
        "version": good[:4] + struct.pack("<H", 2) + good[6:],
        "type": good[:6] + b"\x07" + good[7:],
        "header": good[:30],
        "counters": good[:-1],
        "empty": b"",
    }
    for what, data in bad_cases.items():
        with pytest.raises(abi.FormatError) as g:
            native.deserialize_sketch(data)
        with pytest.raises(abi.FormatError) as r:
            ref.deserialize(data)
        assert str(g.value) == str(r.value), what
    # a parameter block the constructor rejects: ConfigError, as Rsra(cfg)
    cfg_bad = good[:7] + struct.pack("<I", 0) + good[11:]
    with pytest.raises(abi.ConfigError):
        native.deserialize_sketch(cfg_bad)


@pytest.mark.gpu
def test_gpu_merges_cpu_node_stream(ora, streams):
    """a GPU node merges a sketch file written by a CPU node (the mixed
    CPU/GPU merge of SURVEY.md §8f-3): equals the oracle's merge"""
    from paper_1805_09246_b200 import native

    name = "small_seed7"
    p = params_of(streams, name)
    cpu_rs = native.deserialize_sketch(bytes(streams[f"{name}__rsra"]))
    cpu_le = native.deserialize_sketch(bytes(streams[f"{name}__slea"]))
    sk = ora.sketch(p)
    rs = native.Rsra(native.rsra_config(p))
    le = native.Slea(native.slea_config(p))
    pool = ora.rng_pair_array(99, 5000)
    for _ in range(int(cpu_rs.slides)):
        rs.slide(); le.slide(); sk.slide()
    native.update_pairs(rs, le, pool)
    sk.update(pool)
    rs.merge_min(cpu_rs)
    le.merge_min(cpu_le)
    _, _, _, _, c_rs = parse(bytes(streams[f"{name}__rsra"]))
    _, _, _, _, c_le = parse(bytes(streams[f"{name}__slea"]))
    ors, ole = sk.cells()
    assert np.array_equal(rs.cells(), np.minimum(ors, c_rs))
    assert np.array_equal(le.cells(), np.minimum(ole, c_le))
