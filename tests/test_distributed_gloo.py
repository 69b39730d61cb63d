"""Multi-rank merge protocol on CPU (torch.distributed, gloo, world_size 2).

The GPU engine's distributed mode (srlg_engine_set_merge)
merges one edge-router stream per rank: each rank marks the cells its records
touched in the current slice in a u8 map, the maps are max-reduced onto the
root, and the root sets those cells to "recorded this slice" before the
per-slide detection. This test runs exactly that protocol with the CPU
oracle standing in for each rank's device scan and gloo standing in for
NCCL, and checks it against the single-node reference semantics
(run_distributed, src/distributed.cpp:35-117): the root's sketches are
bit-exact with a single node fed the whole trace after every slice, and the
root's reports are byte-identical with the single-node engine's.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_09246_b200 import abi, synth

WORLD = 2


def mix64(x):
    x = x.astype(np.uint64)
    x ^= x >> np.uint64(30)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(27)
    x *= np.uint64(0x94D049BB133111EB)
    x ^= x >> np.uint64(31)
    return x


def route_hash_pair(pairs, nodes):
    """route() policy hash_pair (src/distributed.cpp:22-24)."""
    key = (pairs["aip"].astype(np.uint64) << np.uint64(32)) | pairs["bip"].astype(np.uint64)
    seed_mix = mix64(np.array([0x70617274], dtype=np.uint64))[0]
    with np.errstate(over="ignore"):
        h = mix64(seed_mix + key * np.uint64(0x9E3779B97F4A7C15))
    return (h % np.uint64(nodes)).astype(np.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle import oracle as O

        ora = O.backend("ora")
        w = synth.scaled(synth.WORKLOADS["c2"], packets=240_000, n_slices=8, planted=12,
                         planted_spread=4, bg_hosts=20_000)
        params = abi.small_params(11)
        k = 3
        pairs, off = synth.trace(w).generate()
        local = ora.sketch(params)  # this rank's own stream
        root_global = ora.sketch(params) if rank == 0 else None
        whole = ora.sketch(params) if rank == 0 else None
        blobs = []
        wc = abi.WindowConfig(k=k, theta=64)
        n_slices = len(off) - 1
        for s in range(n_slices):
            chunk = pairs[off[s]: off[s + 1]]
            mine = chunk[route_hash_pair(chunk, WORLD) == rank]
            local.update(mine)
            rs, le = local.cells()
            # touched in this slice <=> distance 0 after the updates
            marks = torch.from_numpy(np.concatenate([(rs == 0), (le == 0)]).astype(np.uint8))
            dist.reduce(marks, dst=0, op=dist.ReduceOp.MAX)
            if rank == 0:
                g_rs, g_le = root_global.cells()
                m = marks.numpy().astype(bool)
                g_rs[m[: len(g_rs)]] = 0
                g_le[m[len(g_rs):]] = 0
                root_global.set_cells(g_rs, g_le)
                whole.update(chunk)
                w_rs, w_le = whole.cells()
                assert np.array_equal(g_rs, w_rs), f"rsra diverged at slice {s}"
                assert np.array_equal(g_le, w_le), f"slea diverged at slice {s}"
                last = s == n_slices - 1
                if s + 1 >= k or last:
                    blobs.append(root_global.detect(wc, s, partial=last))
                if not last:
                    root_global.slide()
                    whole.slide()
            local.slide()
        if rank == 0:
            e = ora.engine(params, abi.WindowConfig(k=k, theta=64, t0_us=0))
            e.process_slices(pairs, off)
            e.finish()
            result_q.put(("ok", b"".join(blobs) == e.take_reports(), len(blobs)))
    except Exception as exc:  # surface failures to the parent
        result_q.put(("error", repr(exc), rank))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_merge_protocol_equals_single_node():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = []
    while not q.empty():
        results.append(q.get())
    assert all(p.exitcode == 0 for p in procs), results
    ok = [r for r in results if r[0] == "ok"]
    assert ok and ok[0][1], results
    assert ok[0][2] >= 6
