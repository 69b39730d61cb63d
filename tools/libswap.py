"""Tools only: SRLG_TOOLS_LIB=path makes the diagnostics scripts load another
build of libsrlg.so (A/B of two builds on one box); symbols the build lacks
read as no-ops."""
import ctypes as C
import os
from pathlib import Path

from paper_1805_09246_b200 import native


class _Tolerant(C.CDLL):
    def __getattr__(self, name):
        try:
            return super().__getattr__(name)
        except AttributeError:
            if name.startswith("__"):
                raise

            def missing(*a):
                return 0

            setattr(self, name, missing)
            return missing


if os.environ.get("SRLG_TOOLS_LIB"):
    native.C.CDLL = _Tolerant
    native.LIB_PATH = Path(os.environ["SRLG_TOOLS_LIB"]).resolve()
