"""ctypes binding of the C ABI (include/srlg.h, built to _lib/libsrlg.so).

The classes mirror the reference's estimator API — `Rsra`, `Slea`,
`run_detection`, `WindowEngine` (proj/core/include/slidecard/*.hpp) — with the
same argument meaning and the same exception types (abi.py). There is no CPU
fallback: importing the library fails loudly when it is missing, and every
call fails with DeviceError when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import abi

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libsrlg.so"

_P = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32
_i = C.c_int
_lib = None


def lib() -> C.CDLL:
    """Load libsrlg.so; raise if the CUDA extension has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    L = C.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL)

    def sig(name, res, *args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = list(args)

    R, S, E = _P, _P, _P
    sig("srlg_last_error", C.c_char_p)
    sig("srlg_abi_version", _i)
    sig("srlg_kernel_launches", _u64)
    sig("srlg_device_count", _i, C.POINTER(_i))
    sig("srlg_params_validate", _i, C.POINTER(abi.Params))
    sig("srlg_params_rsra_config", _i, C.POINTER(abi.Params), C.POINTER(abi.RsraConfig))
    sig("srlg_params_slea_config", _i, C.POINTER(abi.Params), C.POINTER(abi.SleaConfig))
    sig("srlg_slea_row_length_for", _u64, C.POINTER(abi.SleaConfig))
    sig("srlg_window_config_validate", _i, C.POINTER(abi.WindowConfig))
    sig("srlg_rsra_create", _i, C.POINTER(abi.RsraConfig), _i, C.POINTER(_P))
    sig("srlg_rsra_clone", _i, R, C.POINTER(_P))
    sig("srlg_rsra_serialized_size", _u64, R)
    sig("srlg_slea_serialized_size", _u64, S)
    sig("srlg_rsra_serialize", _i, R, _P, _u64, C.POINTER(_u64))
    sig("srlg_slea_serialize", _i, S, _P, _u64, C.POINTER(_u64))
    sig("srlg_deserialize_sketch", _i, _P, _u64, _i, C.POINTER(_i), C.POINTER(_P), C.POINTER(_P),
        C.POINTER(_u64))
    sig("srlg_rsra_config_get", _i, R, C.POINTER(abi.RsraConfig))
    sig("srlg_slea_config_get", _i, S, C.POINTER(abi.SleaConfig))
    sig("srlg_rsra_destroy", None, R)
    sig("srlg_rsra_num_cells", _u64, R)
    sig("srlg_rsra_slides", _u64, R)
    sig("srlg_rsra_set_slides", _i, R, _u64)
    sig("srlg_rsra_slide", _i, R)
    sig("srlg_rsra_reinitialize", _i, R)
    sig("srlg_rsra_extract_hot", _i, R, _u32, _P, _u64, _P)
    sig("srlg_rsra_export_cells", _i, R, _P, _u64)
    sig("srlg_rsra_import_cells", _i, R, _P, _u64)
    sig("srlg_rsra_export_stamps", _i, R, _P, _u64, C.POINTER(_u32), C.POINTER(_u32))
    sig("srlg_rsra_compatibility_mismatch", _i, R, R, C.c_char_p, C.c_size_t)
    sig("srlg_rsra_merge_min", _i, R, R)
    sig("srlg_rsra_forward", _i, R, _u32, _P)
    sig("srlg_rsra_device_ptr", _P, R)
    sig("srlg_slea_create", _i, C.POINTER(abi.SleaConfig), _i, C.POINTER(_P))
    sig("srlg_slea_clone", _i, S, C.POINTER(_P))
    sig("srlg_slea_destroy", None, S)
    sig("srlg_slea_num_cells", _u64, S)
    sig("srlg_slea_row_length", _u64, S)
    sig("srlg_slea_slides", _u64, S)
    sig("srlg_slea_set_slides", _i, S, _u64)
    sig("srlg_slea_slide", _i, S)
    sig("srlg_slea_reinitialize", _i, S)
    sig("srlg_slea_row_weights", _i, S, _u32, _P)
    sig("srlg_slea_estimate_context", _i, S, _u32, _P, C.POINTER(C.c_double))
    sig("srlg_slea_usle_weights", _i, S, _u32, _P, _u64, _P)
    sig("srlg_slea_estimate", _i, S, _u32, _u32, C.c_double, C.POINTER(abi.Estimate))
    sig("srlg_slea_lh_column", _i, S, _u32, _u32, C.POINTER(_u32))
    sig("srlg_slea_export_cells", _i, S, _P, _u64)
    sig("srlg_slea_import_cells", _i, S, _P, _u64)
    sig("srlg_slea_export_stamps", _i, S, _P, _u64, C.POINTER(_u32), C.POINTER(_u32))
    sig("srlg_slea_compatibility_mismatch", _i, S, S, C.c_char_p, C.c_size_t)
    sig("srlg_slea_merge_min", _i, S, S)
    sig("srlg_slea_device_ptr", _P, S)
    sig("srlg_update_pairs", _i, R, S, _P, _u64, _i, _P)
    sig("srlg_reconstruct", _i, R, _P, _P, _u64, _u64, _P, _u64, C.POINTER(_u64), C.POINTER(_i),
        C.POINTER(_u64), C.POINTER(_u64))
    sig("srlg_detect", _i, R, S, C.POINTER(abi.WindowConfig), _u64, _i, _P, _u64,
        C.POINTER(_u64))
    sig("srlg_engine_create", _i, C.POINTER(abi.WindowConfig), R, S, C.POINTER(_P))
    sig("srlg_engine_destroy", None, E)
    sig("srlg_engine_process", _i, E, _P, _u64)
    sig("srlg_engine_process_slices", _i, E, _P, _P, _u64, _u64, _i)
    sig("srlg_engine_advance_to_slice", _i, E, _u64)
    sig("srlg_engine_finish", _i, E)
    sig("srlg_engine_sync", _i, E)
    sig("srlg_engine_take_reports", _i, E, _P, _u64, C.POINTER(_u64), C.POINTER(_u64))
    sig("srlg_engine_current_slice", _u64, E)
    sig("srlg_engine_records", _u64, E)
    sig("srlg_engine_clamped", _u64, E)
    sig("srlg_engine_rsra", _P, E)
    sig("srlg_engine_slea", _P, E)
    sig("srlg_engine_reset", _i, E)
    sig("srlg_engine_kernel_launches", _u64, E)
    sig("srlg_nccl_unique_id", _i, _P)
    sig("srlg_nccl_comm_create", _i, _i, _P, _i, _i, C.POINTER(_P))
    sig("srlg_nccl_comm_destroy", _i, _P)
    sig("srlg_engine_set_merge", _i, E, _P, _i, _i, _i)
    sig("srlg_engine_merge_stats", _i, E, C.POINTER(_u64), C.POINTER(_u64))
    sig("srlg_engine_merge_create", _i, E, _i, _u64, _P)
    sig("srlg_engine_merge_join", _i, E, _i, _P)
    sig("srlg_engine_merge_attach", _i, E, _i, E)
    sig("srlg_lane_create", _i, _i, _i, C.POINTER(_i))
    sig("srlg_profile_read_engine", _i, _i, C.POINTER(C.c_double), C.POINTER(_u64),
        C.POINTER(_u64))
    sig("srlg_engine_detect_latency", _i, E, C.POINTER(C.c_double), C.POINTER(_u64))
    sig("srlg_engine_set_persistent", _i, E, _i)
    sig("srlg_engine_set_arena", _i, E, _u64)
    sig("srlg_engine_set_incremental", _i, E, _i)
    sig("srlg_engine_inc_stats", _i, E, C.POINTER(_u64))
    sig("srlg_engine_set_recon", _i, E, _i, _i)
    sig("srlg_engine_set_anet", _i, E, C.POINTER(abi.Anet))
    sig("srlg_exact_create", _i, _u64, _u32, _u64, _i, C.POINTER(_P))
    sig("srlg_exact_destroy", None, _P)
    sig("srlg_exact_process_slices", _i, _P, _P, _P, _u64, _u64, _i)
    sig("srlg_exact_finish", _i, _P)
    sig("srlg_exact_distinct_pairs", _u64, _P)
    sig("srlg_exact_take_windows", _i, _P, _P, _u64, C.POINTER(_u64), C.POINTER(_u64))
    sig("srlg_engine_process_file", _i, E, C.c_char_p, C.POINTER(_u64))
    sig("srlg_update_raw", _i, R, S, _P, _u64, _i, C.POINTER(abi.Anet), C.POINTER(_u64))
    sig("srlg_engine_trace_ops", _i, E, _i)
    sig("srlg_engine_detect_phases", _i, E, C.POINTER(C.c_double))
    sig("srlg_engine_detect_diag", _i, E, C.POINTER(C.c_double))
    sig("srlg_engine_read_io_trace", _i, E, C.POINTER(C.c_float), _u64, C.POINTER(_u64))
    sig("srlg_engine_read_cta_trace", _i, E, C.POINTER(_u64), _u64, C.POINTER(_u64),
        C.POINTER(_u64))
    sig("srlg_engine_read_op_trace", _i, E, C.POINTER(_u64), _u64, C.POINTER(_u64))
    sig("srlg_device_stream", _P, _i)
    sig("srlg_profile_enable", _i, _i, _i)
    sig("srlg_profile_read", _i, _i, C.POINTER(C.c_double), C.POINTER(_u64), C.POINTER(_u64),
        C.POINTER(C.c_double), C.POINTER(_u64))
    sig("srlg_io_bytes", _i, _i, C.POINTER(_u64), C.POINTER(_u64))
    sig("srlg_detect_phase_ns", _i, _i, _P)
    sig("srlg_bench_random_updates", _i, _i, _u64, _u64, _i, _i, C.POINTER(C.c_double))
    sig("srlg_bench_trace_updates", _i, R, S, _P, _u64, _i, C.POINTER(C.c_double), C.POINTER(_u64))
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != abi.OK:
        abi.raise_for(rc, lib().srlg_last_error().decode())


def device_count() -> int:
    n = _i()
    check(lib().srlg_device_count(C.byref(n)))
    return n.value


def kernel_launches() -> int:
    return lib().srlg_kernel_launches()


def rsra_config(params: abi.Params) -> abi.RsraConfig:
    c = abi.RsraConfig()
    check(lib().srlg_params_rsra_config(C.byref(params), C.byref(c)))
    return c


def slea_config(params: abi.Params) -> abi.SleaConfig:
    c = abi.SleaConfig()
    check(lib().srlg_params_slea_config(C.byref(params), C.byref(c)))
    return c


def validate(params: abi.Params) -> None:
    check(lib().srlg_params_validate(C.byref(params)))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class _Handle:
    _destroy = ""

    def __init__(self, h, owned=True):
        self.h = h
        self.owned = owned

    def __del__(self):
        if getattr(self, "h", None) and self.owned and _lib is not None:
            getattr(_lib, self._destroy)(self.h)
        self.h = None


class Rsra(_Handle):
    """Device-backed Rsra (include/slidecard/rsra.hpp:29-77)."""

    _destroy = "srlg_rsra_destroy"

    def __init__(self, cfg: abi.RsraConfig | None = None, device: int = 0, _h=None,
                 owned=True):
        if _h is None:
            p = _P()
            check(lib().srlg_rsra_create(C.byref(cfg), device, C.byref(p)))
            _h = p.value
        super().__init__(_h, owned)
        self.cfg = abi.RsraConfig()
        check(lib().srlg_rsra_config_get(self.h, C.byref(self.cfg)))

    def clone(self) -> "Rsra":
        p = _P()
        check(lib().srlg_rsra_clone(self.h, C.byref(p)))
        return Rsra(_h=p.value)

    @property
    def num_cells(self) -> int:
        return lib().srlg_rsra_num_cells(self.h)

    @property
    def slides(self) -> int:
        return lib().srlg_rsra_slides(self.h)

    def set_slides(self, s: int) -> None:
        check(lib().srlg_rsra_set_slides(self.h, s))

    def slide(self) -> None:
        check(lib().srlg_rsra_slide(self.h))

    def reinitialize(self) -> None:
        check(lib().srlg_rsra_reinitialize(self.h))

    def update(self, pairs: np.ndarray) -> None:
        update_pairs(self, None, pairs)

    def extract_hot(self, k: int) -> list[np.ndarray]:
        cap = max(1, self.cfg.r << self.cfg.q)
        cols = np.zeros(cap, dtype=np.uint32)
        counts = np.zeros(self.cfg.r, dtype=np.uint64)
        check(lib().srlg_rsra_extract_hot(self.h, k, _ptr(cols), cap, _ptr(counts)))
        out, off = [], 0
        for c in counts:
            out.append(cols[off: off + int(c)].copy())
            off += int(c)
        return out

    def cells(self) -> np.ndarray:
        out = np.zeros(self.num_cells, dtype=np.uint16)
        check(lib().srlg_rsra_export_cells(self.h, _ptr(out), len(out)))
        return out

    def set_cells(self, cells: np.ndarray) -> None:
        a = np.ascontiguousarray(cells, dtype=np.uint16)
        check(lib().srlg_rsra_import_cells(self.h, _ptr(a), len(a)))

    def stamps(self):
        out = np.zeros(self.num_cells, dtype=np.uint32)
        now, floor = _u32(), _u32()
        check(lib().srlg_rsra_export_stamps(self.h, _ptr(out), len(out), C.byref(now),
                                            C.byref(floor)))
        return out, now.value, floor.value

    def serialize(self) -> bytes:
        """serialize_sketch (sketch_io.cpp:106-119): the "SRLG" v1 stream"""
        n = lib().srlg_rsra_serialized_size(self.h)
        buf = (C.c_uint8 * n)()
        w = _u64(0)
        check(lib().srlg_rsra_serialize(self.h, buf, n, C.byref(w)))
        return bytes(buf)

    def compatibility_mismatch(self, other: "Rsra") -> str:
        buf = C.create_string_buffer(128)
        check(lib().srlg_rsra_compatibility_mismatch(self.h, other.h, buf, 128))
        return buf.value.decode()

    def merge_min(self, other: "Rsra") -> None:
        check(lib().srlg_rsra_merge_min(self.h, other.h))

    def forward(self, aip: int) -> np.ndarray:
        out = np.zeros(self.cfg.r, dtype=np.uint32)
        check(lib().srlg_rsra_forward(self.h, aip, _ptr(out)))
        return out


class Slea(_Handle):
    """Device-backed Slea (include/slidecard/slea.hpp:29-100)."""

    _destroy = "srlg_slea_destroy"

    def __init__(self, cfg: abi.SleaConfig | None = None, device: int = 0, _h=None,
                 owned=True):
        if _h is None:
            p = _P()
            check(lib().srlg_slea_create(C.byref(cfg), device, C.byref(p)))
            _h = p.value
        super().__init__(_h, owned)
        self.cfg = abi.SleaConfig()
        check(lib().srlg_slea_config_get(self.h, C.byref(self.cfg)))

    def clone(self) -> "Slea":
        p = _P()
        check(lib().srlg_slea_clone(self.h, C.byref(p)))
        return Slea(_h=p.value)

    @property
    def num_cells(self) -> int:
        return lib().srlg_slea_num_cells(self.h)

    @property
    def row_length(self) -> int:
        return lib().srlg_slea_row_length(self.h)

    @property
    def slides(self) -> int:
        return lib().srlg_slea_slides(self.h)

    def set_slides(self, s: int) -> None:
        check(lib().srlg_slea_set_slides(self.h, s))

    def slide(self) -> None:
        check(lib().srlg_slea_slide(self.h))

    def reinitialize(self) -> None:
        check(lib().srlg_slea_reinitialize(self.h))

    def update(self, pairs: np.ndarray) -> None:
        update_pairs(None, self, pairs)

    def row_weights(self, k: int) -> np.ndarray:
        out = np.zeros(self.cfg.r, dtype=np.uint64)
        check(lib().srlg_slea_row_weights(self.h, k, _ptr(out)))
        return out

    def estimate_context(self, k: int):
        f = np.zeros(self.cfg.r, dtype=np.float64)
        sfp = C.c_double()
        check(lib().srlg_slea_estimate_context(self.h, k, _ptr(f), C.byref(sfp)))
        return f, sfp.value

    def usle_weights(self, k: int, aips) -> np.ndarray:
        a = np.ascontiguousarray(aips, dtype=np.uint32)
        out = np.zeros(len(a), dtype=np.uint64)
        check(lib().srlg_slea_usle_weights(self.h, k, _ptr(a), len(a), _ptr(out)))
        return out

    def estimate(self, aip: int, k: int, sf_product: float | None = None) -> abi.Estimate:
        if sf_product is None:
            sf_product = self.estimate_context(k)[1]
        e = abi.Estimate()
        check(lib().srlg_slea_estimate(self.h, aip, k, sf_product, C.byref(e)))
        return e

    def lh_column(self, row: int, aip: int) -> int:
        v = _u32()
        check(lib().srlg_slea_lh_column(self.h, row, aip, C.byref(v)))
        return v.value

    def cells(self) -> np.ndarray:
        out = np.zeros(self.num_cells, dtype=np.uint16)
        check(lib().srlg_slea_export_cells(self.h, _ptr(out), len(out)))
        return out

    def set_cells(self, cells: np.ndarray) -> None:
        a = np.ascontiguousarray(cells, dtype=np.uint16)
        check(lib().srlg_slea_import_cells(self.h, _ptr(a), len(a)))

    def stamps(self):
        out = np.zeros(self.num_cells, dtype=np.uint32)
        now, floor = _u32(), _u32()
        check(lib().srlg_slea_export_stamps(self.h, _ptr(out), len(out), C.byref(now),
                                            C.byref(floor)))
        return out, now.value, floor.value

    def serialize(self) -> bytes:
        """serialize_sketch (sketch_io.cpp:121-134): the "SRLG" v1 stream"""
        n = lib().srlg_slea_serialized_size(self.h)
        buf = (C.c_uint8 * n)()
        w = _u64(0)
        check(lib().srlg_slea_serialize(self.h, buf, n, C.byref(w)))
        return bytes(buf)

    def compatibility_mismatch(self, other: "Slea") -> str:
        buf = C.create_string_buffer(128)
        check(lib().srlg_slea_compatibility_mismatch(self.h, other.h, buf, 128))
        return buf.value.decode()

    def merge_min(self, other: "Slea") -> None:
        check(lib().srlg_slea_merge_min(self.h, other.h))


def deserialize_sketch(data: bytes, device: int = 0):
    """deserialize_sketch (sketch_io.cpp:144-175): an "SRLG" v1 stream -> a
    new device-backed Rsra or Slea; FormatError-class failures raise with
    SRLG_ERR_FORMAT"""
    buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
    t, r, s_, used = _i(0), _P(), _P(), _u64(0)
    check(lib().srlg_deserialize_sketch(buf, len(data), device, C.byref(t), C.byref(r),
                                        C.byref(s_), C.byref(used)))
    return Rsra(_h=r.value) if t.value == 1 else Slea(_h=s_.value)


def update_pairs(rsra: Rsra | None, slea: Slea | None, pairs=None, *, device_ptr: int = 0,
                 n: int = 0, stream: int = 0) -> None:
    """Rsra::update + Slea::update over a batch (host numpy pairs, or a device
    pointer to n interleaved {aip, bip} u32 pairs)."""
    r = rsra.h if rsra is not None else None
    s = slea.h if slea is not None else None
    if device_ptr:
        check(lib().srlg_update_pairs(r, s, device_ptr, n, 1, stream or None))
    else:
        a = np.ascontiguousarray(pairs, dtype=abi.PAIR_DTYPE)
        check(lib().srlg_update_pairs(r, s, _ptr(a), len(a), 0, None))


def update_raw(rsra: Rsra | None, slea: Slea | None, packets, anet: abi.Anet) -> int:
    """classify (trace.cpp:111-116) fused into the scan: raw packets
    {src, dst} (PAIR_DTYPE, aip = src, bip = dst) -> records produced"""
    a = np.ascontiguousarray(packets, dtype=abi.PAIR_DTYPE)
    n = _u64(0)
    check(lib().srlg_update_raw(rsra.h if rsra is not None else None,
                                slea.h if slea is not None else None, _ptr(a), len(a), 0,
                                C.byref(anet), C.byref(n)))
    return n.value


def reconstruct(rsra: Rsra, hot_lists, tuple_cap: int = 1 << 22, work_cap: int = 1 << 32):
    counts = np.array([len(h) for h in hot_lists], dtype=np.uint64)
    flat = (np.concatenate([np.asarray(h, dtype=np.uint32) for h in hot_lists])
            if len(hot_lists) else np.zeros(0, np.uint32))
    flat = np.ascontiguousarray(flat, dtype=np.uint32)
    if flat.size == 0:
        flat = np.zeros(1, np.uint32)
    cap = 1 << 20
    out = np.zeros(cap, dtype=np.uint32)
    n, ov, ch, kp = _u64(), _i(), _u64(), _u64()
    check(lib().srlg_reconstruct(rsra.h, _ptr(flat), _ptr(counts), tuple_cap, work_cap, _ptr(out),
                                 cap, C.byref(n), C.byref(ov), C.byref(ch), C.byref(kp)))
    return dict(addresses=out[: n.value].copy(), overflow=bool(ov.value),
                tuples_checked=ch.value, tuples_kept=kp.value)


def run_detection(rsra: Rsra, slea: Slea, wcfg: abi.WindowConfig, window_end: int,
                  partial: bool = False) -> bytes:
    """run_detection (src/window.cpp:36-78) -> one report blob."""
    cap = 1 << 24
    buf = np.zeros(cap, dtype=np.uint8)
    n = _u64()
    check(lib().srlg_detect(rsra.h, slea.h, C.byref(wcfg), window_end, int(partial), _ptr(buf),
                            cap, C.byref(n)))
    return bytes(buf[: n.value])


class WindowEngine(_Handle):
    """WindowEngine (include/slidecard/window.hpp:64-98); takes ownership of
    both sketches like the reference's by-value constructor."""

    _destroy = "srlg_engine_destroy"

    def __init__(self, wcfg: abi.WindowConfig, rsra: Rsra, slea: Slea):
        p = _P()
        check(lib().srlg_engine_create(C.byref(wcfg), rsra.h, slea.h, C.byref(p)))
        rsra.owned = False
        slea.owned = False
        super().__init__(p.value)
        self.wcfg = wcfg
        self._rsra = Rsra(_h=lib().srlg_engine_rsra(self.h), owned=False)
        self._slea = Slea(_h=lib().srlg_engine_slea(self.h), owned=False)

    @classmethod
    def from_params(cls, params: abi.Params, wcfg: abi.WindowConfig, device: int = 0):
        return cls(wcfg, Rsra(rsra_config(params), device), Slea(slea_config(params), device))

    def rsra(self) -> Rsra:
        return self._rsra

    def slea(self) -> Slea:
        return self._slea

    def process(self, records: np.ndarray) -> None:
        recs = np.ascontiguousarray(records, dtype=abi.RECORD_DTYPE)
        check(lib().srlg_engine_process(self.h, _ptr(recs), len(recs)))

    def process_slices(self, pairs=None, offsets=None, first_slice: int = 0, *,
                       device_ptr: int = 0) -> None:
        offs = np.ascontiguousarray(offsets, dtype=np.uint64)
        if device_ptr:
            check(lib().srlg_engine_process_slices(self.h, device_ptr, _ptr(offs), len(offs) - 1,
                                                   first_slice, 1))
        else:
            a = pairs if isinstance(pairs, np.ndarray) and pairs.flags.c_contiguous else \
                np.ascontiguousarray(pairs, dtype=abi.PAIR_DTYPE)
            check(lib().srlg_engine_process_slices(self.h, _ptr(a) if not isinstance(a, int) else a,
                                                   _ptr(offs), len(offs) - 1, first_slice, 0))

    def process_slices_host_ptr(self, host_ptr: int, offsets, first_slice: int = 0) -> None:
        offs = np.ascontiguousarray(offsets, dtype=np.uint64)
        check(lib().srlg_engine_process_slices(self.h, host_ptr, _ptr(offs), len(offs) - 1,
                                               first_slice, 0))

    def advance_to_slice(self, s: int) -> None:
        check(lib().srlg_engine_advance_to_slice(self.h, s))

    def finish(self) -> None:
        check(lib().srlg_engine_finish(self.h))

    def sync(self) -> None:
        check(lib().srlg_engine_sync(self.h))

    def reset(self) -> None:
        check(lib().srlg_engine_reset(self.h))

    def take_reports(self) -> bytes:
        need, nr = _u64(), _u64()
        check(lib().srlg_engine_take_reports(self.h, None, 0, C.byref(need), C.byref(nr)))
        buf = np.zeros(max(1, need.value), dtype=np.uint8)
        check(lib().srlg_engine_take_reports(self.h, _ptr(buf), len(buf), C.byref(need),
                                             C.byref(nr)))
        return bytes(buf[: need.value])

    @property
    def current_slice(self) -> int:
        return lib().srlg_engine_current_slice(self.h)

    @property
    def records(self) -> int:
        return lib().srlg_engine_records(self.h)

    @property
    def clamped(self) -> int:
        return lib().srlg_engine_clamped(self.h)

    def kernel_launches(self) -> int:
        return lib().srlg_engine_kernel_launches(self.h)

    def set_merge(self, comm: int, rank: int, nranks: int, root: int = 0) -> None:
        """Distributed mode: this rank's stream is merged onto `root` every
        slide (NCCL max-reduce of touched-cell maps); only the root reports."""
        check(lib().srlg_engine_set_merge(self.h, comm, rank, nranks, root))

    def process_file(self, path) -> int:
        """binary trace file of 16 B {ts, aip|src, bip|dst} records"""
        n = _u64(0)
        check(lib().srlg_engine_process_file(self.h, str(path).encode(), C.byref(n)))
        return n.value

    def set_anet(self, anet: abi.Anet | None) -> None:
        """raw-packet ingest for later process_slices calls (None: records)"""
        check(lib().srlg_engine_set_anet(self.h, C.byref(anet) if anet is not None else None))

    def set_arena(self, entries: int) -> None:
        """capacity of the ring of candidates past each window's first 1024
        (0 = default)"""
        check(lib().srlg_engine_set_arena(self.h, entries))

    def set_incremental(self, mode: int) -> None:
        """Persistent batches track the window incrementally (a launch's
        first detection sweeps the state, later ones only the blocks that
        changed): 1 (default) the RSRA always and the SLEA when it exceeds
        64 MiB, 2 both always, 3 the RSRA only, 0 off (every detection
        sweeps)."""
        check(lib().srlg_engine_set_incremental(self.h, int(mode)))

    def set_recon(self, ctas: int = 0, groups: int = 0) -> None:
        """reconstruction pipeline: CTAs and groups (0 keeps a value)"""
        check(lib().srlg_engine_set_recon(self.h, ctas, groups))

    def inc_stats(self) -> tuple[int, int]:
        """diagnostics: (RSRA, SLEA) blocks re-examined by incremental
        detections since the last call (counted while trace_ops is on)"""
        out = (_u64 * 4)()
        check(lib().srlg_engine_inc_stats(self.h, out))
        return int(out[0]), int(out[1])

    def set_persistent(self, on: bool) -> None:
        """True (default): pre-sliced runs execute as one persistent kernel
        per batch; False: a scan and a detection launch per slice."""
        check(lib().srlg_engine_set_persistent(self.h, int(on)))

    def trace_ops(self, on: bool) -> None:
        """diagnostics: record the device span of every op of later persistent
        batches"""
        check(lib().srlg_engine_trace_ops(self.h, int(on)))

    def read_op_trace(self) -> np.ndarray:
        """(n, 3) u64 rows {kind (0 scan, 1 detect), start ns, end ns}"""
        n = _u64(0)
        check(lib().srlg_engine_read_op_trace(self.h, None, 0, C.byref(n)))
        out = np.zeros((n.value, 3), dtype=np.uint64)
        if n.value:
            check(lib().srlg_engine_read_op_trace(self.h, out.ctypes.data_as(C.POINTER(_u64)),
                                                  n.value, C.byref(n)))
        return out

    def detect_phases(self) -> dict:
        """mean µs per detection phase since the last call (CTA 0's view);
        call before detect_latency()"""
        out = (C.c_double * 6)()
        check(lib().srlg_engine_detect_phases(self.h, out))
        return dict(zip(("A1_hot", "barrier1", "B_recon_A2_slea", "barrier2", "C_usle",
                         "epilogue"), (round(x, 2) for x in out)))

    def detect_diag(self) -> dict:
        """means per traced detection (see srlg_engine_detect_diag)"""
        o = (C.c_double * 16)()
        check(lib().srlg_engine_detect_diag(self.h, o))
        return {"dfs_end_us": round(o[0], 2), "a2_end_us": round(o[1], 2),
                "dfs_warps_per_cta": round(o[2], 1), "invert_end_us": round(o[3], 2),
                "hot_per_row": [round(x, 1) for x in o[4:9]], "candidates": round(o[12], 1),
                "complete_tuples": round(o[13], 1), "detections": int(o[14])}

    def read_cta_trace(self) -> np.ndarray:
        """(ops, grid, 8) u64 ns per CTA of the last traced batch: op start, A1 done,
        barrier 1 passed, B/A2 done, barrier 2 passed, C done, epilogue done, op end
        (detect ops; scan ops fill 0 and 7 only)"""
        n, g = _u64(0), _u64(0)
        check(lib().srlg_engine_read_cta_trace(self.h, None, 0, C.byref(n), C.byref(g)))
        out = np.zeros((n.value, g.value, 21), dtype=np.uint64)
        check(lib().srlg_engine_read_cta_trace(self.h, out.ctypes.data_as(C.POINTER(_u64)),
                                               out.size, C.byref(n), C.byref(g)))
        return out

    def read_io_trace(self) -> np.ndarray:
        """ms of each chunk copy done, then of each batch launch (last traced
        resident-input run)"""
        n = _u64(0)
        check(lib().srlg_engine_read_io_trace(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.float32)
        check(lib().srlg_engine_read_io_trace(self.h, out.ctypes.data_as(C.POINTER(C.c_float)),
                                              n.value, C.byref(n)))
        return out

    def detect_latency(self):
        """(mean device µs per detection, windows) of persistent batches since
        the last call."""
        us, n = C.c_double(), _u64()
        check(lib().srlg_engine_detect_latency(self.h, C.byref(us), C.byref(n)))
        return us.value, n.value

    def merge_create(self, nranks: int, max_pairs_per_slice: int) -> bytes:
        """In-engine merge: this engine becomes rank 0 (the root) of a group
        of `nranks`; returns the inbox's IPC handle for ranks in other
        processes (srlg_engine_merge_create)."""
        buf = (C.c_uint8 * 64)()
        check(lib().srlg_engine_merge_create(self.h, nranks, max_pairs_per_slice, buf))
        return bytes(buf)

    def merge_join(self, rank: int, ipc_handle: bytes) -> None:
        """join as sending rank `rank` through the root's IPC handle"""
        buf = (C.c_uint8 * 64).from_buffer_copy(ipc_handle)
        check(lib().srlg_engine_merge_join(self.h, rank, buf))

    def merge_attach(self, rank: int, root: "WindowEngine") -> None:
        """join as sending rank `rank` of a root engine in this process"""
        check(lib().srlg_engine_merge_attach(self.h, rank, root.h))

    def merge_stats(self):
        m, b = _u64(), _u64()
        check(lib().srlg_engine_merge_stats(self.h, C.byref(m), C.byref(b)))
        return dict(slice_merges=m.value, bytes_exchanged=b.value)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().srlg_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm_create(nranks: int, uid: bytes, rank: int, device: int) -> int:
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    comm = _P()
    check(lib().srlg_nccl_comm_create(nranks, buf, rank, device, C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    check(lib().srlg_nccl_comm_destroy(comm))


def lane_create(device: int = 0, ctas: int = 0) -> int:
    """A further execution lane on `device` (own streams, persistent kernels
    of at most `ctas` CTAs); returns a device ordinal for Rsra / Slea /
    WindowEngine.from_params."""
    d = _i()
    check(lib().srlg_lane_create(device, ctas, C.byref(d)))
    return d.value


def device_stream(device: int = 0) -> int:
    """cudaStream_t (as int) of the library's compute stream on `device`."""
    return lib().srlg_device_stream(device) or 0


def profile_enable(device: int, on: bool) -> None:
    check(lib().srlg_profile_enable(device, int(on)))


def profile_read(device: int = 0) -> dict:
    sm, sl, sp, dm, dw = C.c_double(), _u64(), _u64(), C.c_double(), _u64()
    check(lib().srlg_profile_read(device, C.byref(sm), C.byref(sl), C.byref(sp), C.byref(dm),
                                  C.byref(dw)))
    return dict(scan_ms=sm.value, scan_launches=sl.value, scan_pairs=sp.value,
                detect_ms=dm.value, detect_windows=dw.value)


def profile_read_engine(device: int = 0) -> dict:
    ms, n, p = C.c_double(), _u64(), _u64()
    check(lib().srlg_profile_read_engine(device, C.byref(ms), C.byref(n), C.byref(p)))
    return dict(engine_ms=ms.value, engine_launches=n.value, engine_pairs=p.value)


def io_bytes(device: int = 0):
    h, d = _u64(), _u64()
    check(lib().srlg_io_bytes(device, C.byref(h), C.byref(d)))
    return h.value, d.value


def bench_random_updates(device: int, n_cells: int, n_updates: int, mode: int = 0,
                         reps: int = 5) -> float:
    r = C.c_double()
    check(lib().srlg_bench_random_updates(device, n_cells, n_updates, mode, reps, C.byref(r)))
    return r.value


def bench_trace_updates(rsra: Rsra, slea: Slea, device_ptr: int, n: int, reps: int = 3):
    """(updates/s, updates per replay): red.max replay of the cell-index
    stream of n device-resident pairs (the random-update roofline on the
    trace's own address distribution)"""
    r, k = C.c_double(), _u64()
    check(lib().srlg_bench_trace_updates(rsra.h, slea.h, device_ptr, n, reps, C.byref(r),
                                         C.byref(k)))
    return r.value, k.value


def detect_phase_ns(device: int = 0) -> dict:
    """Phase durations (ns) of the last fused detection on `device`."""
    t = np.zeros(16, dtype=np.uint64).astype(np.int64)
    check(lib().srlg_detect_phase_ns(device, t.ctypes.data))
    names = ["counts", "barrier1", "reconstruct", "barrier2", "usle", "epilogue"]
    out = {n: int(t[i + 1] - t[i]) for i, n in enumerate(names)}
    out["stages_rel_ns"] = [int(x - t[2]) if x else None for x in t[8:16]]
    return out


class ExactOracle(_Handle):
    """ExactSlidingOracle (exact_oracle.hpp:25-62) on the device: exact
    per-window super points for scoring."""

    _destroy = "srlg_exact_destroy"

    def __init__(self, theta: int = 1024, k: int = 300, max_pairs: int = 100_000_000,
                 device: int = 0):
        p = _P()
        check(lib().srlg_exact_create(theta, k, max_pairs, device, C.byref(p)))
        super().__init__(p.value)

    def process_slices(self, pairs=None, offsets=None, first_slice: int = 0, *,
                       device_ptr: int = 0) -> None:
        offs = np.ascontiguousarray(offsets, dtype=np.uint64)
        if device_ptr:
            check(lib().srlg_exact_process_slices(self.h, device_ptr, _ptr(offs), len(offs) - 1,
                                                  first_slice, 1))
        else:
            a = np.ascontiguousarray(pairs, dtype=abi.PAIR_DTYPE)
            check(lib().srlg_exact_process_slices(self.h, _ptr(a), _ptr(offs), len(offs) - 1,
                                                  first_slice, 0))

    def finish(self) -> None:
        check(lib().srlg_exact_finish(self.h))

    @property
    def distinct_pairs(self) -> int:
        return lib().srlg_exact_distinct_pairs(self.h)

    def take_windows(self) -> bytes:
        n, w = _u64(0), _u64(0)
        check(lib().srlg_exact_take_windows(self.h, None, 0, C.byref(n), C.byref(w)))
        buf = (C.c_uint8 * max(1, n.value))()
        check(lib().srlg_exact_take_windows(self.h, buf, n.value, C.byref(n), C.byref(w)))
        return bytes(buf)[: n.value]
