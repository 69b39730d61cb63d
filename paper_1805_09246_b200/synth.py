"""Deterministic synthetic edge-router traffic (csrc/synth.c) and the
workload presets of SURVEY.md §8d. Input generation only — not the path."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import abi

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libsrlg_synth.so")
_lib = None


class Spec(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("n_slices", C.c_uint64), ("packets", C.c_uint64),
        ("bg_hosts", C.c_uint64), ("bg_zipf", C.c_double), ("bg_card_exp", C.c_double),
        ("bg_max_card", C.c_uint32), ("planted", C.c_uint32), ("planted_min", C.c_uint32),
        ("planted_max", C.c_uint32), ("planted_spread", C.c_uint32), ("reserved", C.c_uint32),
        ("ddos_sources", C.c_uint64),
    ]


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing; run the build")
        L = C.CDLL(_LIB_PATH)
        L.srlg_synth_create.restype = C.c_void_p
        L.srlg_synth_create.argtypes = [C.POINTER(Spec)]
        L.srlg_synth_destroy.argtypes = [C.c_void_p]
        L.srlg_synth_offsets.restype = C.c_uint64
        L.srlg_synth_offsets.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.srlg_synth_generate.restype = C.c_int
        L.srlg_synth_generate.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                          C.c_void_p, C.c_uint32]
        L.srlg_synth_planted_aip.restype = C.c_uint32
        L.srlg_synth_planted_aip.argtypes = [C.c_void_p, C.c_uint64]
        L.srlg_synth_planted_card.restype = C.c_uint32
        L.srlg_synth_planted_card.argtypes = [C.c_void_p, C.c_uint64]
        L.srlg_synth_victim_aip.restype = C.c_uint32
        L.srlg_synth_victim_aip.argtypes = [C.c_void_p]
        _lib = L
    return _lib


@dataclass
class Workload:
    """A named synthetic configuration plus the sketch/window parameters it is
    measured with."""

    name: str
    spec: dict
    params: dict
    k: int
    reinit: bool = False

    def sketch_params(self) -> abi.Params:
        return abi.Params(**self.params)

    def window_config(self, **kw) -> abi.WindowConfig:
        d = dict(k=self.k, theta=self.params.get("theta", 1024), t0_us=0,
                 reinit_per_window=int(self.reinit))
        d.update(kw)
        return abi.WindowConfig(**d)


class Trace:
    def __init__(self, **spec):
        self.spec = Spec(**spec)
        self.h = _L().srlg_synth_create(C.byref(self.spec))
        if not self.h:
            raise ValueError("bad synth spec")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.srlg_synth_destroy(self.h)
            self.h = None

    @property
    def n_slices(self) -> int:
        return self.spec.n_slices

    def offsets(self, first: int = 0, n: int | None = None) -> np.ndarray:
        n = self.spec.n_slices - first if n is None else n
        off = np.zeros(n + 1, dtype=np.uint64)
        _L().srlg_synth_offsets(self.h, first, n, off.ctypes.data)
        return off

    def generate(self, first: int = 0, n: int | None = None, threads: int | None = None,
                 out: np.ndarray | None = None):
        """pairs (structured aip/bip array) + slice offsets for slices
        first .. first+n-1. `out` may be a preallocated (e.g. pinned) buffer."""
        off = self.offsets(first, n)
        total = int(off[-1])
        if out is None:
            out = np.empty(total, dtype=abi.PAIR_DTYPE)
        assert len(out) >= total
        threads = threads or min(64, os.cpu_count() or 1)
        _L().srlg_synth_generate(self.h, first, len(off) - 1, off.ctypes.data, out.ctypes.data,
                                 threads)
        return out[:total], off

    def planted(self):
        return [(_L().srlg_synth_planted_aip(self.h, p), _L().srlg_synth_planted_card(self.h, p))
                for p in range(self.spec.planted)]

    def victim_aip(self) -> int:
        return _L().srlg_synth_victim_aip(self.h)


DEFAULT_PARAMS = dict(q=17, r=5, delta=5, eta=8, q_prime=17, r_prime=5, delta_prime=16,
                      eta_prime=16384, theta=1024, seed=808)

WORKLOADS = {
    # C1: discrete window (k=1, strict reinit), 2^20 packets, 100 planted supers
    "c1": Workload("c1_discrete_1slice_2^20", dict(
        seed=2025, n_slices=1, packets=1 << 20, bg_hosts=500_000, bg_zipf=0.5, bg_card_exp=0.5,
        bg_max_card=511, planted=100, planted_min=2048, planted_max=4096, planted_spread=1),
        DEFAULT_PARAMS, k=1, reinit=True),
    # C2: sliding window k=300 over 600 slices, 100M packets, Zipf(1.0) hosts
    "c2": Workload("c2_sliding_k300_600slices_100M_zipf", dict(
        seed=2025, n_slices=600, packets=100_000_000, bg_hosts=1_000_000, bg_zipf=1.0,
        bg_card_exp=0.5, bg_max_card=511, planted=100, planted_min=2048, planted_max=8192,
        planted_spread=300), DEFAULT_PARAMS, k=300),
    # C4: large SLEA sizing (q'=21, 671 MB of stamps, exceeds L2)
    "c4": Workload("c4_large_qprime21_k300", dict(
        seed=2026, n_slices=600, packets=1_000_000_000, bg_hosts=4_000_000, bg_zipf=1.0,
        bg_card_exp=0.5, bg_max_card=511, planted=100, planted_min=2048, planted_max=8192,
        planted_spread=300), dict(DEFAULT_PARAMS, q_prime=21), k=300),
    # C5: DDoS burst: one victim, 10M distinct sources over uniform background
    "c5": Workload("c5_ddos_10M_sources", dict(
        seed=2027, n_slices=600, packets=100_000_000, bg_hosts=1_000_000, bg_zipf=0.0,
        bg_card_exp=0.0, bg_max_card=2, planted=0, planted_min=0, planted_max=0,
        planted_spread=1, ddos_sources=10_000_000), DEFAULT_PARAMS, k=300),
}


def scaled(w: Workload, packets: int | None = None, n_slices: int | None = None,
           **spec_overrides) -> Workload:
    spec = dict(w.spec)
    if packets is not None:
        spec["packets"] = packets
    if n_slices is not None:
        spec["n_slices"] = n_slices
    spec.update(spec_overrides)
    return Workload(w.name + "_scaled", spec, dict(w.params), w.k, w.reinit)


def trace(w: Workload) -> Trace:
    return Trace(**w.spec)


# ---------------------------------------------------------- edge routers
# route() of run_distributed (src/distributed.cpp:20-31): which node (edge
# router, here: rank) a record lands on. Used to split one synthetic trace
# into per-rank streams.
POLICY_HASH_PAIR, POLICY_ROUND_ROBIN, POLICY_BY_SOURCE_PREFIX = 0, 1, 2


def _mix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def route(pairs: np.ndarray, nodes: int, policy: int = POLICY_HASH_PAIR) -> np.ndarray:
    """node of every record (index = position in the record stream)"""
    if policy == POLICY_HASH_PAIR:  # hash64((aip << 32) | bip, 0x70617274) % nodes
        key = (pairs["aip"].astype(np.uint64) << np.uint64(32)) | pairs["bip"].astype(np.uint64)
        seed = _mix64(np.array([0x70617274], dtype=np.uint64))[0]
        with np.errstate(over="ignore"):
            h = _mix64(seed + key * np.uint64(0x9E3779B97F4A7C15))
        return (h % np.uint64(nodes)).astype(np.int64)
    if policy == POLICY_ROUND_ROBIN:
        return np.arange(len(pairs), dtype=np.int64) % nodes
    if policy == POLICY_BY_SOURCE_PREFIX:
        return (pairs["aip"].astype(np.int64) >> 24) % nodes
    raise ValueError("unknown partition policy")


def split_streams(pairs: np.ndarray, offsets: np.ndarray, nodes: int,
                  policy: int = POLICY_HASH_PAIR):
    """one (pairs, slice offsets) stream per node, every stream with the
    same slices (empty ones included), records in their original order"""
    dest = route(pairs, nodes, policy)
    slice_of = np.repeat(np.arange(len(offsets) - 1), np.diff(offsets.astype(np.int64)))
    out = []
    for n in range(nodes):
        mine = dest == n
        cnt = np.bincount(slice_of[mine], minlength=len(offsets) - 1)
        off = np.zeros(len(offsets), dtype=np.uint64)
        off[1:] = np.cumsum(cnt)
        out.append((np.ascontiguousarray(pairs[mine]), off))
    return out


def records(pairs: np.ndarray, offsets: np.ndarray, slice_us: int, t0_us: int = 0) -> np.ndarray:
    """timestamped records of a pre-sliced trace (each at its slice start)"""
    rec = np.empty(len(pairs), dtype=abi.RECORD_DTYPE)
    slice_of = np.repeat(np.arange(len(offsets) - 1, dtype=np.uint64),
                         np.diff(offsets.astype(np.int64)))
    rec["ts_us"] = np.uint64(t0_us) + slice_of * np.uint64(slice_us)
    rec["aip"] = pairs["aip"]
    rec["bip"] = pairs["bip"]
    return rec
