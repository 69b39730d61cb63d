"""TEST INFRASTRUCTURE ONLY — Python face of the two CPU checkers.

* backend "ora": the plain-C restatement (oracle/srlg_oracle.c,
  built to oracle/_build/libsrlg_oracle.so);
* backend "ref": the unmodified reference library compiled from
  /root/reference by oracle/Makefile (oracle/_ref/libslidecard_ref.so) behind
  the extern "C" shim oracle/ref_shim.cpp.

Both expose the same calls, so tests parametrise over them. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from paper_1805_09246_b200 import abi

HERE = Path(__file__).resolve().parent
LIB_PATHS = {
    "ora": HERE / "_build" / "libsrlg_oracle.so",
    "ref": HERE / "_ref" / "libslidecard_ref.so",
}

_P = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32
_i = C.c_int


def available(kind: str) -> bool:
    return LIB_PATHS[kind].exists()


def build() -> None:
    """Compile the checkers (the reference part only when /root/reference is
    present — it is absent on the GPU box, which uses the prebuilt files)."""
    import subprocess

    targets = ["oracle"]
    if Path("/root/reference/proj/core/src").is_dir():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


class Backend:
    def __init__(self, kind: str):
        if kind not in LIB_PATHS:
            raise ValueError(kind)
        path = LIB_PATHS[kind]
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(str(path), mode=os.RTLD_LOCAL)
        self.p = "ref_" if kind == "ref" else "ora_"
        L, p = self.lib, self.p

        def fn(name, res, *args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = list(args)
            return f

        self.last_error = fn("last_error", C.c_char_p)
        self.mix64 = fn("mix64", _u64, _u64)
        self.hash64 = fn("hash64", _u64, _u64, _u64)
        self.lsb = fn("lsb", _u32, _u32)
        self.sampling_threshold = fn("sampling_threshold", _u32, _u64, _u64)
        self.detection_rho = fn("detection_rho", C.c_double)
        self._le = fn("le_estimate", _i, C.c_double, _u32, C.POINTER(C.c_double), C.POINTER(_i))
        self._cw = fn("corrected_weight", _i, C.c_double, C.c_double, _u32, C.POINTER(C.c_double))
        self._validate = fn("params_validate", _i, C.POINTER(abi.Params))
        self._configs = fn("params_configs", _i, C.POINTER(abi.Params), C.POINTER(abi.RsraConfig),
                           C.POINTER(abi.SleaConfig))
        if kind == "ref":
            self._sk_create = fn("sketch_create", _P, C.POINTER(abi.Params))
            self._en_create = fn("engine_create", _P, C.POINTER(abi.Params),
                                 C.POINTER(abi.WindowConfig))
        else:
            self._sk_create = fn("sketch_create", _P, C.POINTER(abi.RsraConfig),
                                 C.POINTER(abi.SleaConfig))
            self._en_create = fn("engine_create", _P, C.POINTER(abi.RsraConfig),
                                 C.POINTER(abi.SleaConfig), C.POINTER(abi.WindowConfig))
        if kind == "ref":  # the reference's ExactSlidingOracle (exact_oracle.cpp)
            self._exact = fn("exact_detect", _i, _P, _P, _u64, _u64, _u32, _P, _u64,
                             C.POINTER(_u64))
        if kind == "ref":  # the reference's classify (trace.cpp:111-116)
            self._classify = fn("classify", _i, _P, _u64, C.POINTER(abi.Anet), _P,
                                C.POINTER(_u64))
        if kind == "ref":  # the reference's own "SRLG" v1 stream (sketch_io.cpp)
            self._deser = fn("deserialize", _i, _P, _u64, C.POINTER(_i), _P, _u64,
                             C.POINTER(_u64), C.POINTER(_u64))
        self.sk_clone = fn("sketch_clone", _P, _P)
        self.sk_destroy = fn("sketch_destroy", None, _P)
        if kind == "ref":
            self._update = fn("update", _i, _P, _P, _u64, _u32)
        else:
            self._update = fn("update", None, _P, _P, _u64)
        self.update_rsra_only = fn("update_rsra_only", None if kind == "ora" else _i, _P, _P, _u64)
        self.update_slea_only = fn("update_slea_only", None if kind == "ora" else _i, _P, _P, _u64)
        self.slide = fn("slide", None, _P)
        self.reinit = fn("reinit", None, _P)
        self.slides = fn("slides", _u64, _P)
        self.set_slides = fn("set_slides", None, _P, _u64)
        self.rsra_ncells = fn("rsra_ncells", _u64, _P)
        self.slea_ncells = fn("slea_ncells", _u64, _P)
        self.slea_row_length = fn("slea_row_length", _u64, _P)
        self.export = fn("export", None, _P, _P, _P)
        self.import_ = fn("import", None, _P, _P, _P)
        self._merge = fn("merge_min", _i, _P, _P)
        self._hot = fn("extract_hot", _i, _P, _u32, _P, _u64, _P)
        self._ctx = fn("estimate_context", _i, _P, _u32, _P, C.POINTER(C.c_double))
        self._est = fn("estimate", _i, _P, _u32, _u32, C.POINTER(abi.Estimate))
        self.lh_column = fn("lh_column", _u32, _P, _u32, _u32)
        self._fwd = fn("forward", _i, _u32, _u32, _u32, _u64, _u32, _P)
        self._ginfo = fn("group_info", _i, _u32, _u32, _u32, _u64, C.POINTER(_u32), C.POINTER(_i))
        self._inv = fn("invert", _i, _u32, _u32, _u32, _u64, _P, _P, _u64, C.POINTER(_u64))
        self._rec = fn("reconstruct", _i, _u32, _u32, _u32, _u64, _P, _P, _u64, _u64, _u32, _P,
                       _u64, C.POINTER(_u64), C.POINTER(_i), C.POINTER(_u64), C.POINTER(_u64))
        self._detect = fn("detect", _i, _P, C.POINTER(abi.WindowConfig), _u64, _i, _P, _u64,
                          C.POINTER(_u64))
        self.en_destroy = fn("engine_destroy", None, _P)
        self._en_process = fn("engine_process", _i, _P, _P, _u64)
        self._en_slices = fn("engine_process_slices", _i, _P, _P, _P, _u64, _u64)
        self._en_advance = fn("engine_advance", _i, _P, _u64)
        self._en_finish = fn("engine_finish", _i, _P)
        self._en_take = fn("engine_take_reports", _u64, _P, _P, _u64, C.POINTER(_u64))
        self.en_current = fn("engine_current_slice", _u64, _P)
        self.en_export = fn("engine_export", None, _P, _P, _P)
        if kind == "ref":
            self._dist = fn("run_distributed", _i, _P, _u64, C.POINTER(abi.Params),
                            C.POINTER(abi.WindowConfig), _u32, _u32, _P, _u64, C.POINTER(_u64),
                            C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64))
            self.en_clone = fn("engine_clone", _P, _P)
            self.hardware_threads = fn("hardware_threads", C.c_uint)
            self._serialize = fn("serialize", _u64, _P, _i, _P, _u64)
            self._csv = fn("blobs_to_csv", _u64, _P, _u64, _P, _u64)
        else:
            self._dist = fn("run_distributed", _i, _P, _u64, C.POINTER(abi.RsraConfig),
                            C.POINTER(abi.SleaConfig), C.POINTER(abi.WindowConfig), _u32, _u32,
                            _P, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64),
                            C.POINTER(_u64))
            self.fnv1a64_u16 = fn("fnv1a64_u16", _u64, _P, _u64)
        self.rng_pairs = fn("rng_pairs", None, _u64, _u64, _P)

    # ----------------------------------------------------------- helpers
    def check(self, rc: int) -> None:
        if rc != abi.OK:
            abi.raise_for(rc, self.last_error().decode())

    def le_estimate(self, w: float, eta: int):
        v, s = C.c_double(), _i()
        self.check(self._le(w, eta, C.byref(v), C.byref(s)))
        return v.value, bool(s.value)

    def corrected_weight(self, w: float, sfp: float, eta: int) -> float:
        v = C.c_double()
        self.check(self._cw(w, sfp, eta, C.byref(v)))
        return v.value

    def configs(self, params: abi.Params):
        rc, sc = abi.RsraConfig(), abi.SleaConfig()
        self.check(self._configs(C.byref(params), C.byref(rc), C.byref(sc)))
        return rc, sc

    def validate(self, params: abi.Params) -> None:
        self.check(self._validate(C.byref(params)))

    def forward(self, q, r, delta, seed, aip):
        out = np.zeros(r, dtype=np.uint32)
        self.check(self._fwd(q, r, delta, seed, aip, out.ctypes.data))
        return out

    def group_info(self, q, r, delta, seed):
        u, c = _u32(), _i()
        self.check(self._ginfo(q, r, delta, seed, C.byref(u), C.byref(c)))
        return u.value, bool(c.value)

    def invert(self, q, r, delta, seed, cols):
        cols = np.ascontiguousarray(cols, dtype=np.uint32)
        cap = 1 << 12
        out = np.zeros(cap, dtype=np.uint32)
        n = _u64()
        self.check(self._inv(q, r, delta, seed, cols.ctypes.data, out.ctypes.data, cap, C.byref(n)))
        return out[: n.value].copy()

    def reconstruct(self, q, r, delta, seed, hot_lists, tuple_cap=1 << 22, work_cap=1 << 32,
                    workers=1):
        counts = np.array([len(h) for h in hot_lists], dtype=np.uint64)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(h, dtype=np.uint32)
                                                    for h in hot_lists]) if len(hot_lists)
                                    else np.zeros(0, np.uint32), dtype=np.uint32)
        cap = 1 << 20
        out = np.zeros(cap, dtype=np.uint32)
        n, ov, ch, kp = _u64(), _i(), _u64(), _u64()
        self.check(self._rec(q, r, delta, seed, flat.ctypes.data, counts.ctypes.data, tuple_cap,
                             work_cap, workers, out.ctypes.data, cap, C.byref(n), C.byref(ov),
                             C.byref(ch), C.byref(kp)))
        return dict(addresses=out[: n.value].copy(), overflow=bool(ov.value),
                    tuples_checked=ch.value, tuples_kept=kp.value)

    def sketch(self, params: abi.Params) -> "Sketch":
        return Sketch(self, params)

    def exact_detect(self, pairs: np.ndarray, offsets: np.ndarray, theta: int, k: int) -> bytes:
        """reference exact_detect over pre-sliced pairs -> truth-window blob"""
        pairs = np.ascontiguousarray(pairs, dtype=abi.PAIR_DTYPE)
        offs = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = _u64()
        self.check(self._exact(pairs.ctypes.data, offs.ctypes.data, len(offs) - 1, theta, k, None,
                               0, C.byref(n)))
        buf = (C.c_uint8 * max(1, n.value))()
        self.check(self._exact(pairs.ctypes.data, offs.ctypes.data, len(offs) - 1, theta, k, buf,
                               n.value, C.byref(n)))
        return bytes(buf)[: n.value]

    def classify(self, raw: np.ndarray, anet: abi.Anet) -> np.ndarray:
        """reference classify: raw packets (aip = src, bip = dst) -> records"""
        raw = np.ascontiguousarray(raw, dtype=abi.PAIR_DTYPE)
        out = np.zeros(2 * len(raw), dtype=abi.PAIR_DTYPE)
        n = _u64()
        self.check(self._classify(raw.ctypes.data, len(raw), C.byref(anet), out.ctypes.data,
                                  C.byref(n)))
        return out[: n.value].copy()

    def deserialize(self, data: bytes):
        """reference deserialize_sketch: (type 1 rsra / 2 slea, slides, u16 cells)"""
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        t, n, sl = _i(), _u64(), _u64()
        self.check(self._deser(buf, len(data), C.byref(t), None, 0, C.byref(n), C.byref(sl)))
        cells = np.zeros(n.value, dtype=np.uint16)
        self.check(self._deser(buf, len(data), C.byref(t), cells.ctypes.data, n.value, C.byref(n),
                               C.byref(sl)))
        return t.value, sl.value, cells

    def engine(self, params: abi.Params, wcfg: abi.WindowConfig) -> "Engine":
        return Engine(self, params, wcfg)

    def run_distributed(self, records: np.ndarray, params, wcfg, nodes: int, policy: int):
        recs = np.ascontiguousarray(records, dtype=abi.RECORD_DTYPE)
        cap = 1 << 24
        blob = np.zeros(cap, dtype=np.uint8)
        nb, nr, sm, be = _u64(), _u64(), _u64(), _u64()
        if self.kind == "ref":
            rc = self._dist(recs.ctypes.data, len(recs), C.byref(params), C.byref(wcfg), nodes,
                            policy, blob.ctypes.data, cap, C.byref(nb), C.byref(nr), C.byref(sm),
                            C.byref(be))
        else:
            r_cfg, s_cfg = self.configs(params)
            rc = self._dist(recs.ctypes.data, len(recs), C.byref(r_cfg), C.byref(s_cfg),
                            C.byref(wcfg), nodes, policy, blob.ctypes.data, cap, C.byref(nb),
                            C.byref(nr), C.byref(sm), C.byref(be))
        self.check(rc)
        return bytes(blob[: nb.value]), dict(slice_merges=sm.value, bytes_exchanged=be.value)

    def rng_pair_array(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=abi.PAIR_DTYPE)
        self.rng_pairs(seed, n, out.ctypes.data)
        return out


class Sketch:
    """An Rsra + Slea pair on the CPU checker."""

    def __init__(self, be: Backend, params: abi.Params | None = None, _handle=None):
        self.be = be
        if _handle is not None:
            self.h = _handle
        else:
            if be.kind == "ref":
                h = be._sk_create(C.byref(params))
            else:
                rc, sc = be.configs(params)
                h = be._sk_create(C.byref(rc), C.byref(sc))
            if not h:
                abi.raise_for(abi.ERR_CONFIG, be.last_error().decode())
            self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.be.sk_destroy(self.h)
            self.h = None

    def clone(self) -> "Sketch":
        return Sketch(self.be, _handle=self.be.sk_clone(self.h))

    def update(self, pairs: np.ndarray, workers: int = 1) -> None:
        pairs = np.ascontiguousarray(pairs, dtype=abi.PAIR_DTYPE)
        if self.be.kind == "ref":
            self.be.check(self.be._update(self.h, pairs.ctypes.data, len(pairs), workers))
        else:
            self.be._update(self.h, pairs.ctypes.data, len(pairs))

    def slide(self):
        self.be.slide(self.h)

    def reinit(self):
        self.be.reinit(self.h)

    @property
    def slides(self) -> int:
        return self.be.slides(self.h)

    def cells(self):
        rs = np.zeros(self.be.rsra_ncells(self.h), dtype=np.uint16)
        le = np.zeros(self.be.slea_ncells(self.h), dtype=np.uint16)
        self.be.export(self.h, rs.ctypes.data, le.ctypes.data)
        return rs, le

    def set_cells(self, rs=None, le=None):
        rs_p = np.ascontiguousarray(rs, dtype=np.uint16) if rs is not None else None
        le_p = np.ascontiguousarray(le, dtype=np.uint16) if le is not None else None
        self.be.import_(self.h, rs_p.ctypes.data if rs_p is not None else None,
                        le_p.ctypes.data if le_p is not None else None)

    def merge_min(self, other: "Sketch") -> None:
        self.be.check(self.be._merge(self.h, other.h))

    def serialize(self, which: int) -> bytes:
        """reference serialize_sketch of the rsra (1) or slea (2) half"""
        n = self.be._serialize(self.h, which, None, 0)
        buf = (C.c_uint8 * n)()
        self.be._serialize(self.h, which, buf, n)
        return bytes(buf)

    def extract_hot(self, k: int, r: int):
        cap = self.be.rsra_ncells(self.h)
        cols = np.zeros(cap, dtype=np.uint32)
        counts = np.zeros(r, dtype=np.uint64)
        self.be.check(self.be._hot(self.h, k, cols.ctypes.data, cap, counts.ctypes.data))
        out, off = [], 0
        for c in counts:
            out.append(cols[off: off + int(c)].copy())
            off += int(c)
        return out

    def estimate_context(self, k: int, r_prime: int):
        f = np.zeros(r_prime, dtype=np.float64)
        sfp = C.c_double()
        self.be.check(self.be._ctx(self.h, k, f.ctypes.data, C.byref(sfp)))
        return f, sfp.value

    def estimate(self, aip: int, k: int) -> abi.Estimate:
        e = abi.Estimate()
        self.be.check(self.be._est(self.h, aip, k, C.byref(e)))
        return e

    def detect(self, wcfg: abi.WindowConfig, window_end: int, partial: bool = False) -> bytes:
        cap = 1 << 22
        blob = np.zeros(cap, dtype=np.uint8)
        n = _u64()
        self.be.check(self.be._detect(self.h, C.byref(wcfg), window_end, int(partial),
                                      blob.ctypes.data, cap, C.byref(n)))
        return bytes(blob[: n.value])


class Engine:
    """WindowEngine on the CPU checker."""

    def __init__(self, be: Backend, params=None, wcfg=None, _handle=None):
        self.be = be
        if _handle is not None:
            self.h = _handle
            return
        if be.kind == "ref":
            h = be._en_create(C.byref(params), C.byref(wcfg))
        else:
            rc, sc = be.configs(params)
            h = be._en_create(C.byref(rc), C.byref(sc), C.byref(wcfg))
        if not h:
            abi.raise_for(abi.ERR_CONFIG, be.last_error().decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.be.en_destroy(self.h)
            self.h = None

    def clone(self) -> "Engine":
        return Engine(self.be, _handle=self.be.en_clone(self.h))

    def process(self, records: np.ndarray) -> None:
        recs = np.ascontiguousarray(records, dtype=abi.RECORD_DTYPE)
        self.be.check(self.be._en_process(self.h, recs.ctypes.data, len(recs)))

    def process_slices(self, pairs: np.ndarray, offsets: np.ndarray, first_slice: int = 0):
        pairs = np.ascontiguousarray(pairs, dtype=abi.PAIR_DTYPE)
        offs = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.be.check(self.be._en_slices(self.h, pairs.ctypes.data, offs.ctypes.data,
                                         len(offs) - 1, first_slice))

    def advance_to_slice(self, s: int) -> None:
        self.be.check(self.be._en_advance(self.h, s))

    def finish(self) -> None:
        self.be.check(self.be._en_finish(self.h))

    def take_reports(self) -> bytes:
        n = _u64()
        need = self.be._en_take(self.h, None, 0, C.byref(n))
        buf = np.zeros(max(need, 1), dtype=np.uint8)
        got = self.be._en_take(self.h, buf.ctypes.data, len(buf), C.byref(n))
        return bytes(buf[:got])

    @property
    def current_slice(self) -> int:
        return self.be.en_current(self.h)

    def cells(self, rs_n: int, le_n: int):
        rs = np.zeros(rs_n, dtype=np.uint16)
        le = np.zeros(le_n, dtype=np.uint16)
        self.be.en_export(self.h, rs.ctypes.data, le.ctypes.data)
        return rs, le


_CACHE: dict[str, Backend] = {}


def backend(kind: str) -> Backend:
    if kind not in _CACHE:
        _CACHE[kind] = Backend(kind)
    return _CACHE[kind]
