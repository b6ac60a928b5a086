"""Gate fusion into dense k-qubit blocks (BASELINE cfg 4: "30-qubit complex128 variational circuit
with gate fusion into dense 5-qubit blocks (tensor-core path)"; north star subsystem 2).

`fuse_dense(circuit, k)` rewrites a circuit (at its current parameters) as a chain of
put(n, locs => matblock(U)) blocks of at most k qubits.  Greedy, dependency-safe grouping over the
lowered op list (qsim-style): a block absorbs, in program order, every op whose qubits (targets and
controls) fit in the block's k-qubit set and that no earlier still-pending op touches — so every
absorbed op commutes past the ops it overtakes (disjoint qubits).  Each block's 2^k x 2^k matrix
is the ordered product of its ops (numpy, host); on the device a block with 3..5 qubits is ONE
HBM pass on the FP64 tensor cores (dense_mma.cu, DMMA m8n8k4) in complex128.

This is the dense-block alternative to the default tile engine (fused.cu), which keeps every gate
as a 2x2 / 4x4 run inside multi-gate shared-memory tiles.  The two are measured against each other
at 30 qubits in tools/cfg4_dense.py (profiles/r02_cfg4_dense.json): for variational circuits the
densified blocks cost 8 D flops per amplitude (D = 2^k) against ~8 per gate-run for the tile
engine, so the tile engine wins on B200 FP64; dense blocks win for genuinely dense unitaries."""
from __future__ import annotations

import numpy as np

from . import blocks as B
from .sharded import realise_ops
from ._capi import MAT_DENSE, MAT_DIAGONAL, MAT_PERMUTATION


def _op_dense(kind, mat, perm, t, c, f, qubits):
    """Dense matrix of one realised op on the ordered qubit list `qubits` (0-based bit order =
    position in `qubits`; controls included)."""
    d = 1 << len(qubits)
    pos = {q: i for i, q in enumerate(qubits)}
    tgt = [pos[q] for q in t]
    ctl = [(pos[q], v) for q, v in zip(c, f)]
    dt = 1 << len(t)
    if kind == MAT_DIAGONAL:
        m = np.diag(np.asarray(mat, complex))
    elif kind == MAT_PERMUTATION:
        m = np.zeros((dt, dt), complex)
        m[np.arange(dt), np.asarray(perm)] = mat
    else:
        m = np.asarray(mat, complex)
    out = np.zeros((d, d), complex)
    for col in range(d):
        if any(((col >> p) & 1) != v for p, v in ctl):
            out[col, col] = 1.0
            continue
        sub = sum(((col >> p) & 1) << i for i, p in enumerate(tgt))
        base = col
        for p in tgt:
            base &= ~(1 << p)
        for r in range(dt):
            row = base
            for i, p in enumerate(tgt):
                if (r >> i) & 1:
                    row |= 1 << p
            out[row, col] += m[r, sub]
    return out


def dense_blocks(ops, k: int = 5):
    """Groups realised ops (sharded.realise_ops tuples, 1-based qubits) into blocks of <= k qubits.
    Returns [(sorted 1-based qubit tuple, dense matrix)] in application order."""
    pending = list(range(len(ops)))
    out = []
    while pending:
        S: set = set()
        blocked: set = set()
        take, keep = [], []
        for i in pending:
            _, _, _, t, c, _ = ops[i]
            q = set(t) | set(c)
            if q & blocked or len(S | q) > k:
                blocked |= q
                keep.append(i)
            else:
                S |= q
                take.append(i)
        qubits = sorted(S)
        U = np.eye(1 << len(qubits), dtype=complex)
        for i in take:
            U = _op_dense(*ops[i], qubits) @ U
        out.append((tuple(qubits), U))
        pending = keep
    return out


def fuse_dense(circuit: B.Block, k: int = 5) -> B.Block:
    """The circuit at its current parameters as a chain of dense <= k-qubit matblocks."""
    nodes = B.parameter_nodes(circuit)
    em = B._Emitter({id(p): i for i, p in enumerate(nodes)})
    n = circuit.nqubits
    B._lower(circuit, tuple(range(1, n + 1)), (), (), em)
    ops = realise_ops(em, B.parameters(circuit))
    return B.chain(n, *[B.put(n, q, B.matblock(U)) for q, U in dense_blocks(ops, k)])
