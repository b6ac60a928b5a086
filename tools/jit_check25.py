"""Offline (CPU-only) NVRTC build of every specialised kernel of the 25q bench plan:
    QBG_JIT_DUMP=/tmp/d python tools/jit_check25.py   (then cuobjdump -res-usage / -sass /tmp/d/*.cubin)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25
qb.set_qubit_cap(max(30, n))
c = qb.variational_circuit(n, 10)
qb.dispatch(c, "random")
p = qb.compile_block(c)
o = qb.compile_observable(qb.heisenberg(n))
k = ctypes.c_int64()
check(lib().qbg_jit_check(p._h, o._h, 1, 0, ctypes.byref(k)))
print("cubin bytes", k.value)
