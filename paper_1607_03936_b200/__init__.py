"""wbfbt-b200: B200-native FP64 hot path of the weighted-BFBT Stokes
preconditioner (Rudi, Stadler & Ghattas, arXiv 1607.03936).

All arithmetic runs in libwbfbt.so (hand-written sm_100a CUDA).  This package
is a thin ctypes binding over the C ABI of include/wbfbt.h: it marshals torch
CUDA tensors (device memory, streams) and checks arguments.  There is no CPU
fallback: importing without the built library raises.
"""
from ._abi import (WBError, Context, lib, library_path, version, sizes,  # noqa: F401
                   WB_STRICT_LUMP, WB_DEBUG_NOMASK, WB_DEBUG_SCALARS, SYMBOLS)

from .slab import SlabContext, SlabComm, DistComm, ThreadComm  # noqa: F401,E402

__all__ = ["SlabContext", "SlabComm", "DistComm", "ThreadComm", "WBError", "Context", "lib", "library_path", "version", "sizes", "WB_STRICT_LUMP",
           "WB_DEBUG_NOMASK", "WB_DEBUG_SCALARS", "SYMBOLS"]
