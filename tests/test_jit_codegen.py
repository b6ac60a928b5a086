"""The runtime-specialised tile kernels: the host planner runs without a device, and every
kernel it generates compiles with NVRTC for sm_100a (no GPU needed).  CPU only."""
import ctypes
import re

import pytest

import paper_1912_10877_b200 as qb
from paper_1912_10877_b200._capi import check, lib


def test_plan_preview_25q_metric_workload():
    c = qb.variational_circuit(25, 10)
    qb.dispatch(c, "random")
    t = qb.compile_block(c).plan_preview()
    plans = {int(m.group(1)): body for m, body in zip(re.finditer(r"plan dir=(\d)", t), re.split(r"plan dir=\d[^\n]*\n", t)[1:])}
    npass = {d: len(re.findall(r"tile Q=", body)) for d, body in plans.items()}
    # the fusion planner must cover 1025 gates in far fewer passes than gates: forward (0), reverse
    # (2), and the checkpointed pair — reverse (5) and its forward mirror (4, >= one pass per segment)
    assert 0 < npass[0] <= 40 and 0 < npass[2] <= 45, npass
    assert 0 < npass[5] <= 40 and npass[4] >= npass[5], npass
    assert "single gate" not in t  # every gate of the variational circuit tiles
    # every tile holds the three low (coalescing) qubits
    assert all(q.startswith("0,1,2,") for q in re.findall(r"tile Q=([\d,]+)", t))


@pytest.mark.parametrize("n,depth,nb,dtype", [(13, 1, 1, 0), (12, 1, 8, 1)])
def test_generated_kernels_compile_for_sm100a(n, depth, nb, dtype):
    c = qb.variational_circuit(n, depth)
    qb.dispatch(c, "random")
    p = qb.compile_block(c)
    o = qb.compile_observable(qb.heisenberg(n))
    k = ctypes.c_int64()
    check(lib().qbg_jit_check(p._h, o._h, nb, dtype, ctypes.byref(k)))
    assert k.value > 0


def test_generic_gates_plan():
    """Controlled / 2-qubit / multi-qubit diagonal gates all lower to tile ops (no fallbacks)."""
    n = 14
    blocks = [qb.put(n, (3, 9), qb.rot(qb.kron(qb.X, qb.X), 0.3)),
              qb.control(n, (2, -5), 13, qb.shift(0.2)),
              qb.put(n, (1, 14), qb.rot(qb.kron(qb.Z, qb.Z), 0.7)),
              qb.control(n, 7, 8, qb.Ry(0.1)),
              qb.put(n, 4, qb.H)]
    c = qb.chain(n, *blocks)
    p = qb.compile_block(c)
    t = p.plan_preview()
    assert "single gate" not in t
    k = ctypes.c_int64()
    check(lib().qbg_jit_check(p._h, None, 1, 0, ctypes.byref(k)))
    assert k.value > 0


@pytest.mark.parametrize("n,seed", [(12, 3), (14, 11), (13, 19)])
def test_random_circuit_kernels_generate_and_compile(n, seed):
    """Planner invariants (register / thread slots inside the stage layout, checked while the
    kernels are generated) and NVRTC compilation for random circuits over every gate form —
    a CPU-side guard for planner bugs such as a run left off the register slots."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_random_circuits import random_circuit
    c = random_circuit(n, 120, seed)
    p = qb.compile_block(c)
    o = qb.compile_observable(qb.heisenberg(n))
    k = ctypes.c_int64()
    check(lib().qbg_jit_check(p._h, o._h, 1, 0, ctypes.byref(k)))
    assert k.value > 0


def test_folded_checkpoint_plans_25q():
    """Permutation folding: in the checkpointed pair of the 25q/d10 bench workload
    every CNOT of the ring folds into the load / store maps, so each pass holds rotation runs only
    (33 + 33 passes, 77 + 77 stages; 128 + 128 without folding)."""
    c = qb.variational_circuit(25, 10)
    qb.dispatch(c, "random")
    t = qb.compile_block(c).plan_preview()
    for d in (4, 5):
        i = t.index(f"plan dir={d}")
        j = t.find("plan dir", i + 5)
        body = t[i:j if j > 0 else None]
        assert len(re.findall("tile Q", body)) == 33, d
        assert sum(int(x) for x in re.findall(r"stages=(\d+)", body)) <= 80, d
        assert len(re.findall(r"fold=\d+", body)) >= 30, d  # the ring's CNOTs, in (almost) every pass
