"""In-tree build of every native artefact (no JIT cache, so the built .so files
travel to the GPU box with the repo snapshot).

  _lib/libsrlg.so         CUDA kernels (sm_100a) + the C ABI of include/srlg.h
  _lib/libslidecard_b200.so  C++ drop-in of the reference API (include/slidecard/)
  _lib/libsrlg_synth.so   deterministic workload generator (bench/tests input)
  oracle/_build, oracle/_ref   the CPU checkers (test infrastructure)
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_lib"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v"]

CUDA_SRCS = ["kernels.cu", "detect.cu", "capi.cu", "exact.cu"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, quiet=False):
    if not quiet:
        print(" ".join(str(c) for c in cmd), flush=True)
    r = subprocess.run([str(c) for c in cmd], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]}")
    return r


def build_cuda(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libsrlg.so"
    deps = [CSRC / s for s in CUDA_SRCS] + [CSRC / "srlg_internal.cuh", INCLUDE / "srlg.h"]
    if not force and not _stale(out, deps):
        return out
    objs = []
    for s in CUDA_SRCS:
        o = LIB / (Path(s).stem + ".o")
        r = _run([NVCC, *ARCH, *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", CSRC / s, "-o", o])
        # keep the ptxas resource report next to the objects
        (LIB / (Path(s).stem + ".ptxas.txt")).write_text(r.stderr)
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-Xlinker", "-z,defs", "-lcudart_static",
          "-lrt", "-lpthread", "-ldl"])
    return out


def build_synth(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libsrlg_synth.so"
    deps = [CSRC / "synth.c", CSRC / "srlg_synth.h", INCLUDE / "srlg.h"]
    if force or _stale(out, deps):
        _run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-pthread", "-I", INCLUDE, "-I", CSRC,
              "-o", out, CSRC / "synth.c", "-lm"])
    return out


def build_dropin(force: bool = False) -> Path | None:
    src = CSRC / "dropin.cpp"
    if not src.exists():
        return None
    out = LIB / "libslidecard_b200.so"
    hdrs = sorted((INCLUDE / "slidecard").glob("*.hpp"))
    deps = [src, INCLUDE / "srlg.h", *hdrs, LIB / "libsrlg.so"]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-I", INCLUDE,
              "-o", out, src, f"-L{LIB}", "-lsrlg", f"-Wl,-rpath,$ORIGIN"])
    return out


def build_dropin_check(force: bool = False) -> Path | None:
    """tests/cpp/dropin_check: a reference-style caller compiled against the
    drop-in headers (run by tests/test_dropin.py on the GPU)."""
    src = ROOT / "tests" / "cpp" / "dropin_check.cpp"
    out = LIB / "dropin_check"
    lib = LIB / "libslidecard_b200.so"
    if not src.exists() or not lib.exists():
        return None
    hdrs = sorted((INCLUDE / "slidecard").glob("*.hpp"))
    if force or _stale(out, [src, lib, *hdrs]):
        _run(["g++", "-std=c++20", "-O2", "-I", INCLUDE, "-o", out, src, f"-L{LIB}",
              "-lslidecard_b200", "-lsrlg", f"-Wl,-rpath,{LIB}", "-Wl,-rpath,$ORIGIN"])
    return out


REF_TESTS = ["hash", "sliding_counters", "linear_counting", "rsra", "slea", "window",
             "distributed", "sketch_io", "config"]
REF_TEST_DIR = Path("/root/reference/proj/tests")


def build_ref_unit_tests(force: bool = False) -> Path | None:
    """_lib/ref_unit_tests: the reference's own unit tests
    (proj/tests/test_*.cpp, compiled unmodified from where they lie) against
    the drop-in headers, linked to libslidecard_b200 — with the doctest
    stand-in of tests/cpp/doctest_shim. Built here, where /root/reference
    exists; the binary travels to the GPU box like the .so files
    (tests/test_ref_unit_tests.py runs it)."""
    out = LIB / "ref_unit_tests"
    lib = LIB / "libslidecard_b200.so"
    srcs = [REF_TEST_DIR / "doctest_main.cpp"] + [REF_TEST_DIR / f"test_{t}.cpp" for t in REF_TESTS]
    if not lib.exists() or not all(p.exists() for p in srcs):
        return out if out.exists() else None
    shim = ROOT / "tests" / "cpp" / "doctest_shim" / "doctest.h"
    hdrs = sorted((INCLUDE / "slidecard").glob("*.hpp"))
    if not force and not _stale(out, [*srcs, shim, lib, *hdrs]):
        return out
    objdir = LIB / "ref_unit_tests.o"
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in srcs:
        o = objdir / (src.stem + ".o")
        _run(["g++", "-std=c++20", "-O2", "-I", shim.parent, "-I", INCLUDE, "-c", src, "-o", o],
             quiet=True)
        objs.append(o)
    _run(["g++", "-o", out, *objs, f"-L{LIB}", "-lslidecard_b200", "-lsrlg",
          "-Wl,-rpath,$ORIGIN"])
    return out


def build_oracle() -> None:
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as _o  # test infrastructure: builds the checkers only

    _o.build()


def build_all(force: bool = False) -> None:
    build_cuda(force)
    build_synth(force)
    build_dropin(force)
    build_dropin_check(force)
    build_ref_unit_tests(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
