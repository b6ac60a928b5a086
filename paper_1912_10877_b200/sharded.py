"""State vectors sharded across ranks by global qubits.

A state of n qubits is split over G = 2^g ranks: rank r holds the 2^(n-g) amplitudes whose g
"global" physical bits equal r; the other n-g bits are the rank's local register.  A logical ->
physical qubit map lets any logical qubit live in any position.

Per gate (SPEC.md:315-323 semantics, lowered ops):
  * controls on global qubits need no communication: a rank whose bit does not match drops
    the gate, a matching rank drops the control;
  * diagonal gates on global qubits need no communication: the rank's bits select a
    sub-diagonal (or a scalar phase) on the remaining local targets;
  * a non-diagonal target on a global qubit is first SWAPPED with a local qubit: partner ranks
    r and r ^ (1 << k) exchange one half of their local state (the half whose local bit l
    differs from their own global bit k): S_local / 2 per direction per rank (SURVEY §8(e)
    "default: swap"), then the map records the exchange; later gates on that qubit are local.
Expectation values of Pauli sums: terms are grouped by X support, the X support is swapped
local, each rank evaluates its local terms (global Z bits become signs) and the energies are
summed over ranks.

The schedule is host logic independent of where the shards live.  Backends:
  * ``DeviceVirtualBackend``: G shard registers on one GPU, exchanges by device copies (CI for
    the multi-GPU path on one B200; also runs 33-qubit states as 8 x 30-qubit shards);
  * ``DeviceNcclBackend``: one shard per process / GPU, exchanges with NCCL send/recv over
    NVLink through torch.distributed (zero-copy views of the shard registers);
  * tests add a numpy / CPU-oracle backend to check the schedule on CPU (gloo).
All gate arithmetic runs in libqbg (the device backends); the backends only move bytes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import errors
from ._capi import GEN_NONE, GEN_PHASE, GEN_ROTATION, GEN_SHIFT, MAT_DENSE, MAT_DIAGONAL, MAT_IDENTITY, \
    MAT_PERMUTATION


# ---------------------------------------------------------------------------------------------------
# realised local ops
# ---------------------------------------------------------------------------------------------------
@dataclass
class LOp:
    """A realised gate in physical LOCAL positions (0-based) for one rank."""
    kind: int                    # MAT_DIAGONAL / MAT_PERMUTATION / MAT_DENSE
    mat: np.ndarray              # diag (d,), perm vals (d,), dense (d, d) [row, col]
    perm: np.ndarray | None
    targets: tuple               # 0-based local positions, matrix qubit order
    ctrls: tuple = ()
    cfg: tuple = ()


def realise_ops(em, theta) -> list:
    """Lowered program (blocks._Emitter) -> list of (kind, matrix, perm, targets, ctrls, cfg) with
    1-based LOGICAL qubits and matrices realised at theta (gates.hpp:61-92 formulas)."""
    out = []
    vals = np.asarray(em.vals, dtype=complex) if em.vals else np.zeros(0, complex)
    perms = np.asarray(em.perms, dtype=np.int64) if em.perms else np.zeros(0, np.int64)
    for op in em.ops:
        d = op.dim
        t = tuple(op.targets[k] for k in range(op.ntarget))
        c = tuple(op.ctrls[k] for k in range(op.nctrl))
        f = tuple(op.ctrl_cfg[k] for k in range(op.nctrl))
        if op.gen == GEN_SHIFT:
            out.append((MAT_DIAGONAL, np.array([1.0, np.exp(1j * theta[op.param])]), None, t, c, f))
            continue
        if op.gen == GEN_PHASE:
            out.append((MAT_DIAGONAL, np.full(d, np.exp(1j * theta[op.param])), None, t, c, f))
            continue
        if op.kind == MAT_IDENTITY:
            G = np.eye(d, dtype=complex)
            kind, m, p = MAT_DIAGONAL, np.ones(d, complex), None
        elif op.kind == MAT_DIAGONAL:
            kind, m, p = MAT_DIAGONAL, vals[op.data:op.data + d].copy(), None
        elif op.kind == MAT_PERMUTATION:
            kind, m, p = MAT_PERMUTATION, vals[op.data:op.data + d].copy(), perms[op.perm:op.perm + d].copy()
        else:
            kind, m, p = MAT_DENSE, vals[op.data:op.data + d * d].reshape(d, d).T.copy(), None
        if op.gen == GEN_ROTATION:
            th = theta[op.param]
            cth, sth = math.cos(th / 2), math.sin(th / 2)
            if kind == MAT_DIAGONAL:
                m = cth - 1j * sth * m
            else:
                if kind == MAT_PERMUTATION:
                    G = np.zeros((d, d), complex)
                    G[np.arange(d), p] = m
                else:
                    G = m
                kind, m, p = MAT_DENSE, cth * np.eye(d) - 1j * sth * G, None
        out.append((kind, m, p, t, c, f))
    return out


# ---------------------------------------------------------------------------------------------------
# the schedule
# ---------------------------------------------------------------------------------------------------
@dataclass
class QubitMap:
    n: int
    g: int
    phys: list = field(default_factory=list)  # logical (0-based) -> physical position; >= nl means global

    def __post_init__(self):
        if not self.phys:
            self.phys = list(range(self.n))

    @property
    def nl(self):
        return self.n - self.g

    def is_global(self, q):
        return self.phys[q] >= self.nl

    def logical_at(self, pos):
        return self.phys.index(pos)


class ShardedSchedule:
    """Turns realised logical ops into per-rank local op lists and swap steps."""

    def __init__(self, n: int, g: int, lookahead: int = 64):
        if g < 1 or g >= n:
            raise errors.ValidationError("sharded: need 1 <= g < n global qubits")
        self.map = QubitMap(n, g)
        self.lookahead = lookahead

    def _choose_local(self, ops, i, avoid):
        """Local position to swap out: the highest one whose logical qubit is not used soon."""
        m = self.map
        soon = set()
        for (_, _, _, t, c, _) in ops[i:i + self.lookahead]:
            soon.update(q - 1 for q in t)
            soon.update(q - 1 for q in c)
        cands = [p for p in range(m.nl - 1, -1, -1) if m.logical_at(p) not in avoid]
        for p in cands:
            if m.logical_at(p) not in soon:
                return p
        return cands[0]

    def steps(self, ops):
        """Yields ('swap', k, l) and ('ops', [per-op logical tuples]) in order; the per-rank
        specialisation happens in `rank_ops` with the map valid at that point."""
        m = self.map
        seg = []
        for i, op in enumerate(ops):
            kind, mat, perm, t, c, f = op
            if kind != MAT_DIAGONAL:
                need = [q - 1 for q in t if m.is_global(q - 1)]
                if need:
                    if seg:
                        yield ("ops", seg, list(m.phys))
                        seg = []
                    avoid = set(q - 1 for q in t) | set(q - 1 for q in c)
                    for q in need:
                        k = m.phys[q] - m.nl
                        pl = self._choose_local(ops, i, avoid)
                        lq = m.logical_at(pl)
                        m.phys[q], m.phys[lq] = pl, m.nl + k
                        yield ("swap", k, pl)
            seg.append(op)
        if seg:
            yield ("ops", seg, list(m.phys))

    @staticmethod
    def rank_ops(seg, phys, nl, rank) -> list:
        """Specialise a segment of logical ops to one rank (global controls / diagonals resolved)."""
        out = []
        for kind, mat, perm, t, c, f in seg:
            keep = True
            lc, lf = [], []
            for q, v in zip(c, f):
                p = phys[q - 1]
                if p >= nl:
                    if ((rank >> (p - nl)) & 1) != v:
                        keep = False
                        break
                else:
                    lc.append(p)
                    lf.append(v)
            if not keep:
                continue
            tp = [phys[q - 1] for q in t]
            if kind == MAT_DIAGONAL and any(p >= nl for p in tp):
                # fix the global target bits -> sub-diagonal over the local targets
                loc = [k for k, p in enumerate(tp) if p < nl]
                base = 0
                for k, p in enumerate(tp):
                    if p >= nl and (rank >> (p - nl)) & 1:
                        base |= 1 << k
                sub = np.array([mat[base | sum(((j >> a) & 1) << k for a, k in enumerate(loc))]
                                for j in range(1 << len(loc))])
                if loc:
                    out.append(LOp(MAT_DIAGONAL, sub, None, tuple(tp[k] for k in loc), tuple(lc), tuple(lf)))
                else:
                    ph = complex(sub[0])
                    if ph != 1:
                        free = next(p for p in range(nl) if p not in lc)
                        out.append(LOp(MAT_DIAGONAL, np.array([ph, ph]), None, (free,), tuple(lc), tuple(lf)))
                continue
            if any(p >= nl for p in tp):
                raise errors.Error("sharded: non-diagonal target still global (schedule bug)")
            out.append(LOp(kind, mat, perm, tuple(tp), tuple(lc), tuple(lf)))
        return out


# ---------------------------------------------------------------------------------------------------
# executor
# ---------------------------------------------------------------------------------------------------
class ShardedState:
    """n-qubit state over 2^g shards held by `backend` (see module docstring)."""

    def __init__(self, backend, n: int, g: int):
        self.backend = backend
        self.n, self.g = n, g
        self.sched = ShardedSchedule(n, g)

    @property
    def phys(self):
        return self.sched.map.phys

    def apply(self, block, theta=None):
        from .blocks import _Emitter, _lower, parameter_nodes, parameters
        nodes = parameter_nodes(block)
        em = _Emitter({id(p): k for k, p in enumerate(nodes)})
        _lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
        th = parameters(block) if theta is None else np.asarray(theta, float)
        ops = realise_ops(em, th)
        nl = self.n - self.g
        for st in self.sched.steps(ops):
            if st[0] == "swap":
                self.backend.swap(st[1], st[2])
            else:
                _, seg, phys = st
                self.backend.apply_local(lambda r: ShardedSchedule.rank_ops(seg, phys, nl, r))
        return self

    def expect_pauli(self, terms) -> float:
        """Σ_k c_k <ψ|P_k|ψ> for (c, xmask, zmask) over LOGICAL qubits (bit q-1 = qubit q)."""
        nl = self.n - self.g
        m = self.sched.map
        groups = {}
        for c, x, z in terms:
            groups.setdefault(x, []).append((c, x, z))
        total = 0.0
        for x, ts in groups.items():
            glob = [q for q in range(self.n) if (x >> q) & 1 and m.is_global(q)]
            for q in glob:
                k = m.phys[q] - nl
                pl = next(p for p in range(nl - 1, -1, -1) if not (x >> m.logical_at(p)) & 1)
                lq = m.logical_at(pl)
                m.phys[q], m.phys[lq] = pl, nl + k
                self.backend.swap(k, pl)
            phys = list(m.phys)

            def local_terms(r, ts=ts, phys=phys):
                out = []
                for c, xx, zz in ts:
                    xl = zl = 0
                    sgn = 1
                    for q in range(self.n):
                        p = phys[q]
                        if (xx >> q) & 1:
                            xl |= 1 << p
                        if (zz >> q) & 1:
                            if p >= nl:
                                if (r >> (p - nl)) & 1 and not (xx >> q) & 1:
                                    sgn = -sgn
                                elif (xx >> q) & 1:
                                    raise errors.Error("sharded: Y on a global qubit (schedule bug)")
                            else:
                                zl |= 1 << p
                    out.append((c * sgn, xl, zl))
                return out

            total += self.backend.expect_local(local_terms)
        return total

    def state(self) -> np.ndarray:
        """Full logical state (small n): gather the shards and undo the qubit map."""
        shards = self.backend.gather()
        nl = self.n - self.g
        full = np.zeros(1 << self.n, dtype=complex)
        for r, sh in enumerate(shards):
            idx_phys = np.arange(1 << nl, dtype=np.int64) | (r << nl)
            logical = np.zeros_like(idx_phys)
            for q in range(self.n):
                logical |= ((idx_phys >> self.phys[q]) & 1) << q
            full[logical] = sh
        return full


def _half_view(t, nl, l, v):
    """View of the amplitudes whose local bit l == v in a shard viewed as complex pairs."""
    return t.view(1 << (nl - l - 1), 2, 1 << l, 2)[:, v]


class DeviceVirtualBackend:
    """All 2^g shards as libqbg registers on the current GPU; exchanges are device copies."""

    def __init__(self, n: int, g: int, init: str = "zero", seed: int = 42):
        import torch
        from ._capi import check, lib
        from .register import Register
        self.torch = torch
        self.n, self.g, self.nl = n, g, n - g
        check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
        # |0...0>: amplitude 1 on rank 0 (all global bits 0), the other shards are zero
        self.regs = [Register(self.nl, 1, seed) for _ in range(1 << g)]
        check(lib().qbg_set_zero(self.regs[0]._h))
        self.views = [self._view(reg) for reg in self.regs]

    def _view(self, reg):
        return self.torch.as_tensor(_CudaBuf(reg.device_ptr, 2 << self.nl), device="cuda")

    def apply_local(self, rank_ops):
        for r, reg in enumerate(self.regs):
            apply_lops(reg, rank_ops(r))

    def swap(self, k, l):
        for r in range(1 << self.g):
            if (r >> k) & 1:
                continue
            p = r | (1 << k)
            a = _half_view(self.views[r], self.nl, l, 1)   # rank bit 0 sends its l = 1 half
            b = _half_view(self.views[p], self.nl, l, 0)   # partner (bit 1) sends its l = 0 half
            tmp = a.clone()
            a.copy_(b)
            b.copy_(tmp)

    def expect_local(self, local_terms):
        total = 0.0
        for r, reg in enumerate(self.regs):
            total += float(expect_terms(reg, local_terms(r)))
        return total

    def gather(self):
        return [reg.state()[0] for reg in self.regs]


class DeviceNcclBackend:
    """One shard per rank (this process's GPU); exchanges with NCCL over NVLink via
    torch.distributed (zero-copy views of the shard register)."""

    def __init__(self, n: int, g: int, init: str = "zero", seed: int = 42):
        import torch
        import torch.distributed as dist
        from ._capi import check, lib
        from .register import Register
        self.torch, self.dist = torch, dist
        self.n, self.g, self.nl = n, g, n - g
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if self.world != 1 << g:
            raise errors.ValidationError("sharded: world size must be 2^g")
        check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
        self.reg = Register(self.nl, 1, seed)  # zero-filled by qbg_reg_create
        if self.rank == 0:
            check(lib().qbg_set_zero(self.reg._h))
        self.view = torch.as_tensor(_CudaBuf(self.reg.device_ptr, 2 << self.nl), device="cuda")

    def apply_local(self, rank_ops):
        apply_lops(self.reg, rank_ops(self.rank))

    def swap(self, k, l):
        b = (self.rank >> k) & 1
        part = self.rank ^ (1 << k)
        mine = _half_view(self.view, self.nl, l, 1 - b)
        send = mine.contiguous()
        recv = self.torch.empty_like(send)
        ops = [self.dist.P2POp(self.dist.isend, send, part), self.dist.P2POp(self.dist.irecv, recv, part)]
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()
        mine.copy_(recv)

    def expect_local(self, local_terms):
        e = self.torch.tensor([float(expect_terms(self.reg, local_terms(self.rank)))], dtype=self.torch.float64,
                              device="cuda")
        self.dist.all_reduce(e)
        return float(e.item())

    def gather(self):
        out = [self.torch.zeros_like(self.view) for _ in range(self.world)]
        self.dist.all_gather(out, self.view.contiguous())
        return [o.cpu().numpy().view(np.complex128) for o in out]


# ---- helpers ----------------------------------------------------------------------------------------
class _CudaBuf:
    """__cuda_array_interface__ over a raw device pointer (float64 elements)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def lops_program(nqubits: int, lops):
    """A qbg program (constant gates) from realised local ops: the fused engine applies the whole
    segment in tile passes."""
    import ctypes
    from ._capi import QbgOp, check, lib
    ops = (QbgOp * max(1, len(lops)))()
    vals, perms = [], []
    for i, o in enumerate(lops):
        op = ops[i]
        d = 1 << len(o.targets)
        op.kind, op.gen, op.param, op.ntarget, op.nctrl, op.dim = o.kind, GEN_NONE, -1, len(o.targets), len(o.ctrls), d
        for k, t in enumerate(o.targets):
            op.targets[k] = t + 1
        for k, (c, v) in enumerate(zip(o.ctrls, o.cfg)):
            op.ctrls[k] = c + 1
            op.ctrl_cfg[k] = v
        op.data = len(vals)
        op.perm = len(perms)
        if o.kind == MAT_DENSE:
            vals.extend(np.asarray(o.mat, complex).T.reshape(-1))
        else:
            vals.extend(np.asarray(o.mat, complex))
        if o.kind == MAT_PERMUTATION:
            perms.extend(int(p) for p in o.perm)
    v = np.ascontiguousarray(np.array(vals or [0j], dtype=np.complex128))
    p = np.ascontiguousarray(np.array(perms or [0], dtype=np.int64))
    h = ctypes.c_void_p()
    check(lib().qbg_prog_create(nqubits, ops, len(lops), v.ctypes.data, len(vals), p.ctypes.data, len(perms),
                                ctypes.byref(h)))
    return h


def apply_lops(reg, lops):
    """Applies realised local ops to a libqbg register as one fused program."""
    from ._capi import check, lib
    if not lops:
        return
    h = lops_program(reg.nqubits, lops)
    try:
        check(lib().qbg_apply(reg._h, h))
    finally:
        lib().qbg_prog_destroy(h)


def expect_terms(reg, terms) -> float:
    """Re Σ c <ψ|P|ψ> for Pauli terms given as (c, xmask, zmask) over the register's qubits."""
    import ctypes
    from ._capi import QbgPauliTerm, check, lib
    if not terms:
        return 0.0
    arr = (QbgPauliTerm * len(terms))()
    for k, (c, x, z) in enumerate(terms):
        arr[k] = QbgPauliTerm(complex(c).real, complex(c).imag, x, z)
    h = ctypes.c_void_p()
    check(lib().qbg_obs_create(reg.nqubits, arr, len(terms), ctypes.byref(h)))
    try:
        out = np.empty(reg.nbatch)
        check(lib().qbg_expect(reg._h, h, out.ctypes.data))
    finally:
        lib().qbg_obs_destroy(h)
    return float(out.sum())
