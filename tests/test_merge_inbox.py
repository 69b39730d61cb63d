"""In-engine multi-GPU merge (srlg_engine_merge_*; detect.cu rank_scan /
root_apply), run as virtual ranks: N engines on N execution lanes of one
B200, each with its own sketches, stream and CTAs, the ranks publishing their
slices' moved cells into the root's inbox through device memory exactly as
they would over NVLink. The root's reports must be byte-identical with the
reference's own run_distributed (src/distributed.cpp:35-117, oracle/_ref) on
the same records and partition policy, and the root's state bit-exact with a
single reference node fed the whole trace (the merged global).
"""
import numpy as np
import pytest

from paper_1805_09246_b200 import abi, native, synth


def _trace(packets=1_200_000, n_slices=14):
    w = synth.scaled(synth.WORKLOADS["c2"], packets=packets, n_slices=n_slices, planted=25,
                     planted_spread=5)
    pairs, off = synth.trace(w).generate()
    return w, pairs, off


def test_split_streams_partition():
    """the per-rank streams partition every slice, in record order"""
    _, pairs, off = _trace(packets=200_000, n_slices=7)
    for policy in (synth.POLICY_HASH_PAIR, synth.POLICY_ROUND_ROBIN,
                   synth.POLICY_BY_SOURCE_PREFIX):
        streams = synth.split_streams(pairs, off, 3, policy)
        dest = synth.route(pairs, 3, policy)
        for n, (p, o) in enumerate(streams):
            assert len(o) == len(off) and o[-1] == len(p)
            assert np.array_equal(p, pairs[dest == n])
        for j in range(len(off) - 1):
            got = np.concatenate([p[int(o[j]):int(o[j + 1])] for p, o in streams])
            want = pairs[int(off[j]):int(off[j + 1])]
            assert sorted(got.tolist()) == sorted(want.tolist())


def test_route_hash_pair_matches_reference_formula():
    """hash64((aip << 32) | bip, 0x70617274) % nodes (distributed.cpp:22-24),
    checked against the oracle's mix64"""
    from oracle import oracle as O

    ora = O.backend("ora")
    rng = np.random.default_rng(5)
    p = np.zeros(64, dtype=abi.PAIR_DTYPE)
    p["aip"] = rng.integers(0, 2**32, 64, dtype=np.uint64)
    p["bip"] = rng.integers(0, 2**32, 64, dtype=np.uint64)
    got = synth.route(p, 7)
    seed = ora.mix64(0x70617274)
    for i in range(64):
        key = (int(p["aip"][i]) << 32) | int(p["bip"][i])
        h = ora.mix64((seed + key * 0x9E3779B97F4A7C15) & (2**64 - 1))
        assert got[i] == h % 7


def _sms():
    import torch

    return torch.cuda.get_device_properties(0).multi_processor_count


def _run_virtual(w, pairs, off, nranks, wc, policy, host_input=False):
    """root on lane 0 with most CTAs, every other rank on a small lane"""
    import torch

    per = max(4, min(16, _sms() // (2 * nranks)))
    root_lane = native.lane_create(0, _sms() - per * (nranks - 1))
    engines = [native.WindowEngine.from_params(w.sketch_params(), wc, device=root_lane)]
    streams = synth.split_streams(pairs, off, nranks, policy)
    max_pairs = max(int(np.diff(o.astype(np.int64)).max()) for _, o in streams)
    engines[0].merge_create(nranks, max_pairs)
    for r in range(1, nranks):
        e = native.WindowEngine.from_params(w.sketch_params(), wc,
                                            device=native.lane_create(0, per))
        e.merge_attach(r, engines[0])
        engines.append(e)
    bufs = []
    for e, (p, o) in zip(engines, streams):
        if host_input:
            t = torch.empty(max(1, len(p)) * 8, dtype=torch.uint8, pin_memory=True)
            t.numpy()[: len(p) * 8] = p.view(np.uint8)
            bufs.append(t)
        else:
            t = torch.from_numpy(p.view(np.uint8).copy() if len(p) else np.zeros(8, np.uint8))
            bufs.append(t.cuda())
    torch.cuda.synchronize()
    # ranks first: the root's launch then finds every peer already running
    for e, t, (_, o) in list(zip(engines, bufs, streams))[::-1]:
        if host_input:
            e.process_slices_host_ptr(t.data_ptr(), o)
        else:
            e.process_slices(offsets=o, device_ptr=t.data_ptr())
    for e in engines[::-1]:
        e.finish()
    return engines


@pytest.mark.gpu
@pytest.mark.parametrize("nranks,k,reinit,policy", [
    (2, 10, 0, synth.POLICY_HASH_PAIR),
    (4, 10, 0, synth.POLICY_HASH_PAIR),
    (8, 10, 0, synth.POLICY_HASH_PAIR),
    (3, 1, 1, synth.POLICY_ROUND_ROBIN),
    (4, 6, 0, synth.POLICY_BY_SOURCE_PREFIX),  # every record on one rank: empty streams
])
def test_virtual_ranks_vs_reference_run_distributed(ref, nranks, k, reinit, policy):
    w, pairs, off = _trace()
    wc = w.window_config(k=k, t0_us=0, reinit_per_window=reinit)
    expected, st = ref.run_distributed(synth.records(pairs, off, wc.slice_us), w.sketch_params(),
                                       wc, nranks, policy)
    engines = _run_virtual(w, pairs, off, nranks, wc, policy)
    root = engines[0]
    assert root.take_reports() == expected
    for e in engines[1:]:
        assert e.take_reports() == b""
    # the root holds the merged global: one reference node fed everything
    one = ref.engine(w.sketch_params(), wc)
    one.process_slices(pairs, off)
    one.finish()
    rs, le = one.cells(root.rsra().num_cells, root.slea().num_cells)
    assert np.array_equal(root.rsra().cells(), rs)
    assert np.array_equal(root.slea().cells(), le)
    ms = root.merge_stats()
    assert ms["slice_merges"] == len(off) - 1
    assert ms["bytes_exchanged"] > 0 or policy == synth.POLICY_BY_SOURCE_PREFIX


@pytest.mark.gpu
def test_virtual_ranks_host_input_and_repeated_runs(ref):
    """pinned host input (chunk-flagged copies) and a second run after
    reset(): the slice sequence continues across runs"""
    w, pairs, off = _trace(packets=900_000, n_slices=9)
    wc = w.window_config(k=4, t0_us=0)
    expected, _ = ref.run_distributed(synth.records(pairs, off, wc.slice_us), w.sketch_params(),
                                      wc, 3, synth.POLICY_HASH_PAIR)
    engines = _run_virtual(w, pairs, off, 3, wc, synth.POLICY_HASH_PAIR, host_input=True)
    assert engines[0].take_reports() == expected
    import torch

    streams = synth.split_streams(pairs, off, 3)
    for e in engines:
        e.reset()
    bufs = [torch.from_numpy(p.view(np.uint8).copy()).cuda() for p, _ in streams]
    torch.cuda.synchronize()
    for e, t, (_, o) in list(zip(engines, bufs, streams))[::-1]:
        e.process_slices(offsets=o, device_ptr=t.data_ptr())
    for e in engines[::-1]:
        e.finish()
    assert engines[0].take_reports() == expected


@pytest.mark.gpu
def test_merge_setup_errors():
    w, pairs, off = _trace(packets=100_000, n_slices=2)
    wc = w.window_config(k=2, t0_us=0)
    root = native.WindowEngine.from_params(w.sketch_params(), wc)
    with pytest.raises(abi.SrlgError):
        root.merge_create(0, 1000)
    handle = root.merge_create(2, 10)
    assert len(handle) == 64
    other = native.WindowEngine.from_params(w.sketch_params(), wc)
    with pytest.raises(abi.SrlgError):
        other.merge_attach(2, root)  # rank out of range
    with pytest.raises(abi.SrlgError):
        root.process(synth.records(pairs[:10], np.array([0, 10], dtype=np.uint64), 1))
    other.merge_attach(1, root)
    # a slice larger than the inbox was sized for
    with pytest.raises(abi.SrlgError):
        other.process_slices(pairs[:100], np.array([0, 100], dtype=np.uint64))


def _ipc_rank(rank, handle, q, n_slices, policy, nranks):
    """a sending rank in its own process: maps the root's inbox through the
    CUDA IPC handle (srlg_engine_merge_join) and scans its stream"""
    try:
        import torch

        w, pairs, off = _trace(n_slices=n_slices)
        wc = w.window_config(k=6, t0_us=0)
        p, o = synth.split_streams(pairs, off, nranks, policy)[rank]
        e = native.WindowEngine.from_params(w.sketch_params(), wc, device=0)
        e.merge_join(rank, handle)
        d = torch.from_numpy(p.view(np.uint8).copy()).cuda()
        torch.cuda.synchronize()
        e.process_slices(offsets=o, device_ptr=d.data_ptr())
        e.finish()
        q.put((rank, "ok", len(e.take_reports())))
    except Exception as ex:  # reported to the parent
        q.put((rank, repr(ex), -1))


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_ipc_ranks_in_other_processes_vs_reference(ref):
    """the multi-process form bench.py --gpus N runs under torchrun: rank 0's
    engine creates the inbox, ranks 1 and 2 run in their own processes and
    join through the CUDA IPC handle (here on the same GPU: the contexts
    time-slice, so the ranks' and the root's kernels take turns); the root's
    reports byte-identical with the reference's run_distributed"""
    import multiprocessing as mp

    import torch

    nranks, n_slices, policy = 3, 10, synth.POLICY_HASH_PAIR
    w, pairs, off = _trace(n_slices=n_slices)
    wc = w.window_config(k=6, t0_us=0)
    expected, _ = ref.run_distributed(synth.records(pairs, off, wc.slice_us), w.sketch_params(),
                                      wc, nranks, policy)
    streams = synth.split_streams(pairs, off, nranks, policy)
    max_pairs = max(int(np.diff(o.astype(np.int64)).max()) for _, o in streams)
    root = native.WindowEngine.from_params(w.sketch_params(), wc, device=0)
    handle = root.merge_create(nranks, max_pairs)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, handle, q, n_slices, policy, nranks))
             for r in range(1, nranks)]
    for pr in procs:
        pr.start()
    p0, o0 = streams[0]
    d = torch.from_numpy(p0.view(np.uint8).copy()).cuda()
    torch.cuda.synchronize()
    root.process_slices(offsets=o0, device_ptr=d.data_ptr())
    root.finish()
    results = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(r[1] == "ok" and r[2] == 0 for r in results), results
    assert root.take_reports() == expected
    assert root.merge_stats()["slice_merges"] == n_slices
