"""ctypes mirrors of the plain-C types in include/srlg.h.

Only data layouts live here (no library loading), so the product wrapper
(`native.py`) and the test-side oracle wrapper (`oracle/oracle.py`) share one
definition of the boundary's structs and of the report-blob format.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np

MAX_ROWS = 64

# status codes (include/srlg.h, mirrors include/slidecard/errors.hpp:8-53)
OK = 0
ERR_CONFIG = 2
ERR_PARSE = 3
ERR_RESOURCE = 4
ERR_INCOMPATIBLE = 5
ERR_SATURATION = 6
ERR_OUT_OF_RANGE = 7
ERR_INVALID_ARGUMENT = 8
ERR_ORDERING = 9
ERR_FORMAT = 10
ERR_CUDA = 11


class SrlgError(RuntimeError):
    """Base of the Python-side exception mirror of the reference taxonomy."""

    code = -1

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class ConfigError(SrlgError):
    pass


class ParseError(SrlgError):
    pass


class OrderingError(ParseError):
    pass


class FormatError(ParseError):
    pass


class ResourceError(SrlgError):
    pass


class IncompatibleSketchError(SrlgError):
    pass


class SaturationError(SrlgError):
    pass


class OutOfRange(SrlgError, IndexError):
    pass


class InvalidArgument(SrlgError, ValueError):
    pass


class DeviceError(SrlgError):
    pass


_ERRORS = {
    ERR_CONFIG: ConfigError,
    ERR_PARSE: ParseError,
    ERR_RESOURCE: ResourceError,
    ERR_INCOMPATIBLE: IncompatibleSketchError,
    ERR_SATURATION: SaturationError,
    ERR_OUT_OF_RANGE: OutOfRange,
    ERR_INVALID_ARGUMENT: InvalidArgument,
    ERR_ORDERING: OrderingError,
    ERR_FORMAT: FormatError,
    ERR_CUDA: DeviceError,
}


def raise_for(code: int, message: str) -> None:
    if code == OK:
        return
    raise _ERRORS.get(code, SrlgError)(code, message)


class Params(C.Structure):
    """SketchParams (include/slidecard/config.hpp:14-37), paper defaults."""

    _fields_ = [
        ("q", C.c_uint32), ("r", C.c_uint32), ("delta", C.c_uint32), ("eta", C.c_uint32),
        ("q_prime", C.c_uint32), ("r_prime", C.c_uint32), ("delta_prime", C.c_uint32),
        ("eta_prime", C.c_uint32), ("theta", C.c_uint64), ("seed", C.c_uint64),
    ]

    def __init__(self, **kw):
        d = dict(q=17, r=5, delta=5, eta=8, q_prime=17, r_prime=5, delta_prime=16,
                 eta_prime=16384, theta=1024, seed=1)
        d.update(kw)
        super().__init__(**d)

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def small_params(seed: int = 1) -> Params:
    """The reference's small test geometry (tests/test_window.cpp:16-30,
    tests/acceptance/acceptance.cpp:53-67)."""
    return Params(q=12, r=5, delta=7, eta=8, q_prime=8, r_prime=3, delta_prime=8,
                  eta_prime=256, theta=64, seed=seed)


class RsraConfig(C.Structure):
    _fields_ = [
        ("q", C.c_uint32), ("r", C.c_uint32), ("delta", C.c_uint32), ("eta", C.c_uint32),
        ("tau", C.c_uint32), ("reserved", C.c_uint32),
        ("seed_h1", C.c_uint64), ("seed_h2", C.c_uint64), ("seed_rhfg0", C.c_uint64),
    ]


class SleaConfig(C.Structure):
    _fields_ = [
        ("q", C.c_uint32), ("r", C.c_uint32), ("delta", C.c_uint32), ("eta", C.c_uint32),
        ("seed_h3", C.c_uint64), ("seeds_lh", C.c_uint64 * MAX_ROWS),
    ]


class WindowConfig(C.Structure):
    """WindowConfig (include/slidecard/window.hpp:15-26)."""

    _fields_ = [
        ("t0_us", C.c_uint64), ("has_t0", C.c_uint32), ("k", C.c_uint32),
        ("slice_us", C.c_uint64), ("theta", C.c_uint64),
        ("regression_tolerance_us", C.c_uint64), ("tuple_cap", C.c_uint64),
        ("reinit_per_window", C.c_uint32), ("keep_below_threshold", C.c_uint32),
        ("workers", C.c_uint32), ("reserved", C.c_uint32),
    ]

    def __init__(self, **kw):
        d = dict(t0_us=0, has_t0=0, k=300, slice_us=1_000_000, theta=1024,
                 regression_tolerance_us=0, tuple_cap=1 << 22, reinit_per_window=0,
                 keep_below_threshold=0, workers=1)
        t0 = kw.pop("t0_us", None)
        d.update(kw)
        if t0 is not None:
            d["t0_us"] = t0
            d["has_t0"] = 1
        super().__init__(**d)


class Estimate(C.Structure):
    """Slea::Estimate (include/slidecard/slea.hpp:61-67)."""

    _fields_ = [
        ("value", C.c_double), ("corrected_weight", C.c_double),
        ("usle_weight", C.c_uint64), ("sf_product", C.c_double),
        ("saturated", C.c_uint32), ("reserved", C.c_uint32),
    ]


MAX_PREFIXES = 16


class Anet(C.Structure):
    """srlg_anet: AnetSpec (trace.hpp:49-62) as (addr, bits) CIDR prefixes"""

    _fields_ = [("n", C.c_uint32), ("reserved", C.c_uint32),
                ("addr", C.c_uint32 * MAX_PREFIXES), ("bits", C.c_uint32 * MAX_PREFIXES)]

    @classmethod
    def of(cls, prefixes):
        """prefixes: [(addr_u32, bits), ...] or ["a.b.c.d/n", ...]"""
        a = cls()
        a.n = len(prefixes)
        for i, p in enumerate(prefixes):
            if isinstance(p, str):
                ip, bits = p.split("/")
                o = [int(x) for x in ip.split(".")]
                p = ((o[0] << 24) | (o[1] << 16) | (o[2] << 8) | o[3], int(bits))
            a.addr[i], a.bits[i] = p
        return a


PAIR_DTYPE = np.dtype([("aip", "<u4"), ("bip", "<u4")])
RECORD_DTYPE = np.dtype([("ts_us", "<u8"), ("aip", "<u4"), ("bip", "<u4")])

_HDR = struct.Struct("<QQdII BBB 5x")
_ENTRY = struct.Struct("<IId")
assert _HDR.size == 40 and _ENTRY.size == 16


@dataclass
class Report:
    """DetectionReport (include/slidecard/report.hpp:17-27)."""

    window_end_slice: int
    candidate_count: int
    sf_product: float
    partial: bool
    overflow: bool
    slea_saturated: bool
    hot_per_row: list = field(default_factory=list)
    entries: list = field(default_factory=list)  # (aip, estimate, saturated)


def parse_blobs(blob: bytes) -> list[Report]:
    out = []
    off = 0
    n = len(blob)
    while off + _HDR.size <= n:
        (end, cand, sfp, n_rows, n_ent, partial, overflow, sat) = _HDR.unpack_from(blob, off)
        off += _HDR.size
        hot = list(struct.unpack_from(f"<{n_rows}Q", blob, off))
        off += 8 * n_rows
        ents = []
        for _ in range(n_ent):
            aip, s, est = _ENTRY.unpack_from(blob, off)
            off += _ENTRY.size
            ents.append((aip, est, bool(s)))
        out.append(Report(end, cand, sfp, bool(partial), bool(overflow), bool(sat), hot, ents))
    if off != n:
        raise ValueError(f"trailing bytes in report blob ({n - off})")
    return out


def pairs_array(aip, bip) -> np.ndarray:
    a = np.empty(len(aip), dtype=PAIR_DTYPE)
    a["aip"] = aip
    a["bip"] = bip
    return a


def format_ipv4(a: int) -> str:
    return f"{(a >> 24) & 255}.{(a >> 16) & 255}.{(a >> 8) & 255}.{a & 255}"


def reports_to_csv(reports: list[Report]) -> str:
    """report_to_csv (src/report.cpp:35-53): estimate with two decimals."""
    lines = ["window_end_slice,aip,estimate,flags"]
    for r in reports:
        rows = sorted(r.entries, key=lambda e: (-e[1], e[0]))
        for aip, est, sat in rows:
            flags = []
            if r.partial:
                flags.append("partial")
            if sat:
                flags.append("saturated")
            if r.overflow:
                flags.append("overflow")
            lines.append(f"{r.window_end_slice},{format_ipv4(aip)},{est:.2f},{'|'.join(flags)}")
    return "\n".join(lines) + "\n"


def parse_truth(blob: bytes):
    """srlg_exact_take_windows blob -> [(end_slice, partial, [(aip, card), ...])]"""
    import struct

    out, off = [], 0
    while off < len(blob):
        end, partial, n = struct.unpack_from("<QII", blob, off)
        off += 16
        sup = [struct.unpack_from("<IIQ", blob, off + 16 * i) for i in range(n)]
        off += 16 * n
        out.append((end, bool(partial), [(a, c) for a, _, c in sup]))
    return out


def score(detected, truth):
    """score (exact_oracle.cpp:105-132): FPR / FNR / TFR normalised by the
    number of true super points (None when there are none)"""
    det = set(detected)
    tru = {a for a, _ in truth}
    fp = len(det - tru)
    fn = len(tru - det)
    if not tru:
        return dict(n_true=0, n_detected=len(det), fp=fp, fn=fn, fpr=0.0, fnr=0.0, tfr=0.0,
                    defined=False)
    fpr, fnr = fp / len(tru), fn / len(tru)
    return dict(n_true=len(tru), n_detected=len(det), fp=fp, fn=fn, fpr=fpr, fnr=fnr,
                tfr=fpr + fnr, defined=True)
