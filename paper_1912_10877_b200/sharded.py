"""State vectors sharded across ranks by global qubits.

A state of n qubits is split over G = 2^g ranks: rank r holds the 2^(n-g) amplitudes whose g
"global" physical bits equal r; the other n-g bits are the rank's local register.  A logical ->
physical qubit map lets any logical qubit live in any position.

Per gate (SPEC.md:315-323 semantics, lowered ops):
  * controls on global qubits need no communication: a rank whose bit does not match drops
    the gate, a matching rank drops the control;
  * diagonal gates on global qubits need no communication: the rank's bits select a
    sub-diagonal (or a scalar phase) on the remaining local targets;
  * a non-diagonal target on a global qubit must first become local.  The schedule
    (`ShardedSchedule`) treats the local positions as a cache of the qubits the gates touch:
    on a miss it evicts the local qubit whose next non-diagonal use is furthest ahead (Belady's
    rule, over the whole op list) and, in the same exchange, also fetches every other global
    qubit needed before the next-chosen victim would be (up to g pairs per exchange).  One
    exchange of j pairs is an all-to-all inside groups of 2^j ranks: each rank keeps 1/2^j of
    its shard and trades one 1/2^j sub-block with each of its 2^j - 1 partners — (1 - 2^-j) S_local
    per direction, against j/2 S_local for j separate pairwise swaps.
Expectation values of Pauli sums: terms are grouped by X support; the groups are scheduled the
same way (their X support must be local), each rank evaluates its local terms (global Z bits
become signs) and the energies are summed over ranks.

Exchanges are chunked (`ChunkedExchange`): a fixed staging budget (default 2 GiB, two slots of
send + receive buffers per partner) bounds the extra memory to shard + staging, whatever the
shard size — at 36 qubits over 8 GPUs a shard is 128 GiB of a 180 GB B200.  A chunk is packed
from the shard by a libqbg gather kernel (qbg_shard_pack), exchanged with NCCL send/recv through
torch.distributed on the NCCL stream while the next chunk is packed, and scattered back
(qbg_shard_unpack) into the sub-block it came from.

The schedule and the exchange are host logic independent of where the shards live:
  * ``DeviceNcclBackend``: one shard per process / GPU (libqbg register), NCCL transport;
  * ``DeviceVirtualBackend``: 2^g shard registers on one GPU, the same pack / unpack kernels and
    chunk loop with the partner's packed chunk read in place (the single-GPU CI of the path; also
    runs 33-qubit states as 8 x 30-qubit shards);
  * the tests run `DistShardBackend` itself (chunk loop, staging, transport) on gloo with a CPU
    shard that implements only the local pack / unpack / gate primitives.
All gate arithmetic runs in libqbg on the device backends; the exchange only moves bytes.
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


_INF = float("inf")


class ShardedSchedule:
    """Turns realised logical ops into per-rank local op lists and exchange steps.

    Local positions are a cache of logical qubits; the "accesses" are the non-diagonal targets of
    the ops in order (controls and diagonal targets may stay global).  A miss evicts by Belady's
    rule (furthest next access, the whole list known ahead) and prefetches the global qubits that
    are needed before the remaining victims' next access, batching up to g pairs per exchange."""

    def __init__(self, n: int, g: int, min_pos: int = 3):
        if g < 0 or g >= n:
            raise errors.ValidationError("sharded: need 0 <= g < n global qubits")
        self.map = QubitMap(n, g)
        # positions below min_pos (the tile engine's coalescing qubits) are not swapped out while
        # others are available: a victim at position l makes the packed runs 2^l rows long
        self.min_pos = min(min_pos, max(0, n - g - g))
        self.exchanges = []  # [(pairs)] of the steps yielded so far (for reports / tests)

    def reset(self):
        self.map.phys = list(range(self.map.n))

    @staticmethod
    def _accesses(needs):
        """needs: list of sets of logical qubits that must be local at step i -> per-qubit sorted
        step lists (the next-use table)."""
        uses = {}
        for i, s in enumerate(needs):
            for q in s:
                uses.setdefault(q, []).append(i)
        return uses

    @staticmethod
    def _next_use(uses, q, i):
        import bisect
        lst = uses.get(q)
        if not lst:
            return _INF
        k = bisect.bisect_left(lst, i)
        return lst[k] if k < len(lst) else _INF

    def plan_remap(self, needs, uses, i):
        """Pairs (k, l) (global bit, local position) that make needs[i] local at step i."""
        m = self.map
        nl = m.nl
        missing = sorted((q for q in needs[i] if m.is_global(q)), key=lambda q: m.phys[q])
        if not missing:
            return []
        pinned = set(needs[i])

        def victims():
            c = []
            for pos in range(nl):
                lq = m.logical_at(pos)
                if lq in pinned:
                    continue
                c.append((pos >= self.min_pos, self._next_use(uses, lq, i), pos, lq))
            c.sort(key=lambda t: (t[0], t[1], t[2]), reverse=True)  # preferred: high pos, furthest use
            return c

        cand = victims()
        if len(cand) < len(missing):
            raise errors.ValidationError("sharded: an op has more non-diagonal targets than local qubits")
        pairs = []
        chosen = []
        for q in missing:
            v = cand.pop(0)
            chosen.append(v)
            pairs.append((q, v))
        # prefetch: other global qubits whose next access precedes the next victim's
        others = sorted((self._next_use(uses, q, i), q) for q in range(m.n) if m.is_global(q) and q not in missing)
        for nu, q in others:
            if len(pairs) >= m.g or not cand or nu == _INF:
                break
            if nu < cand[0][1]:
                pairs.append((q, cand.pop(0)))
        out = []
        for q, (_, _, pos, lq) in pairs:
            k = m.phys[q] - nl
            m.phys[q], m.phys[lq] = pos, nl + k
            out.append((k, pos))
        self.exchanges.append(out)
        return out

    def steps(self, ops):
        """Yields ('remap', [(k, l), ...]) and ('ops', [logical ops], phys) in order; the per-rank
        specialisation happens in `rank_ops` with the map valid at that point."""
        needs = [set(q - 1 for q in t) if kind != MAT_DIAGONAL else set() for (kind, _, _, t, _, _) in ops]
        uses = self._accesses(needs)
        m = self.map
        seg = []
        for i, op in enumerate(ops):
            if any(m.is_global(q) for q in needs[i]):
                if seg:
                    yield ("ops", seg, list(m.phys))
                    seg = []
                yield ("remap", self.plan_remap(needs, uses, i))
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
        self._ops_cache = {}

    @property
    def phys(self):
        return self.sched.map.phys

    def reset_zero(self):
        """|0...0>: every qubit map describes it, so the map returns to the identity too."""
        self.backend.set_zero()
        self.sched.reset()
        return self

    def _realised(self, block, theta):
        from .blocks import _Emitter, _lower, parameter_nodes, parameters
        cached = self._ops_cache.get("block")
        if cached is block:  # identity, not id(): a freed block's id can be reused
            em = self._ops_cache["em"]
        else:
            nodes = parameter_nodes(block)
            em = _Emitter({id(p): k for k, p in enumerate(nodes)})
            _lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
            self._ops_cache = {"block": block, "em": em}
        th = parameters(block) if theta is None else np.asarray(theta, float)
        return realise_ops(em, th)

    def apply(self, block, theta=None):
        ops = self._realised(block, theta)
        nl = self.n - self.g
        for st in self.sched.steps(ops):
            if st[0] == "remap":
                self.backend.remap(st[1])
            else:
                _, seg, phys = st
                self.backend.apply_local(lambda r, seg=seg, phys=phys: ShardedSchedule.rank_ops(seg, phys, nl, r))
        return self

    def expect_pauli(self, terms) -> float:
        """Σ_k c_k <ψ|P_k|ψ> for (c, xmask, zmask) over LOGICAL qubits (bit q-1 = qubit q)."""
        nl = self.n - self.g
        m = self.sched.map
        groups = {}
        for c, x, z in terms:
            groups.setdefault(x, []).append((c, x, z))
        # order: groups already local first, then by the schedule (Belady over the X supports)
        order = sorted(groups, key=lambda x: sum(1 for q in range(self.n) if (x >> q) & 1 and m.is_global(q)))
        needs = [set(q for q in range(self.n) if (x >> q) & 1) for x in order]
        uses = ShardedSchedule._accesses(needs)
        total = 0.0
        batch = []  # local-term builders of the groups evaluated together (one fused seed pass set)

        def flush():
            nonlocal total, batch
            if batch:
                fns = batch
                total += self.backend.expect_local(lambda r: [t for f in fns for t in f(r)])
                batch = []

        for i, x in enumerate(order):
            if any(m.is_global(q) for q in needs[i]):
                flush()
                self.backend.remap(self.sched.plan_remap(needs, uses, i))
            phys = list(m.phys)

            def local_terms(r, ts=groups[x], phys=phys):
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

            batch.append(local_terms)
        flush()
        return self.backend.reduce_sum(total)

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


# ---------------------------------------------------------------------------------------------------
# chunked exchange
# ---------------------------------------------------------------------------------------------------
DEFAULT_STAGING_BYTES = 2 << 30


def remap_groups(rank: int, pairs):
    """For a remap of pairs (k_i, l_i): the partners of `rank` and, per partner, the fixed local
    positions and their values selecting the sub-block traded with it (the partner's k-bits)."""
    ks = [k for k, _ in pairs]
    ls = [l for _, l in pairs]
    mine = sum(((rank >> k) & 1) << i for i, k in enumerate(ks))
    out = []
    for pat in range(1 << len(pairs)):
        if pat == mine:
            continue
        prank = rank
        for i, k in enumerate(ks):
            prank = (prank & ~(1 << k)) | (((pat >> i) & 1) << k)
        out.append((prank, ls, pat))
    return out


class ChunkedExchange:
    """The chunk loop of a remap, shared by the backends.  `local` provides rows_per_shard,
    row_bytes, arena(nbytes) (a flat staging buffer of 8-byte words, allocated once),
    pack(ls, pat, row0, nrows, buf) and unpack(ls, pat, row0, nrows, buf); `transport` provides
    start(sends, recvs, peers, nbytes) -> handle and finish(handle).  The staging arena holds two
    slots of (send, receive) chunk buffers per partner.  Per chunk: pack for every partner, post
    the transfers, then — while the next chunk is packed into the other slot — wait for the
    previous chunk and unpack it.  Extra memory: the arena, nothing else."""

    def __init__(self, local, transport, rank: int, staging_bytes: int = DEFAULT_STAGING_BYTES):
        self.local, self.transport, self.rank = local, transport, rank
        self.staging_bytes = int(staging_bytes)
        self.bytes_sent = 0
        self.chunks = 0
        self.events = None  # a list: every remap appends its (start, end) CUDA events (measurement)

    def chunk_rows(self, npartners):
        per = self.staging_bytes // (2 * 2 * npartners)  # 2 slots x (send + recv) per partner
        rows = max(1, per // self.local.row_bytes)
        return 1 << (rows.bit_length() - 1)  # power of two: chunks tile the sub-block evenly

    def remap(self, pairs):
        if not pairs:
            return
        groups = remap_groups(self.rank, pairs)
        sub_rows = self.local.rows_per_shard >> len(pairs)
        cr = min(sub_rows, self.chunk_rows(len(groups)))
        words = cr * self.local.row_bytes // 8
        arena = self.local.arena(4 * len(groups) * words * 8)
        slots = [[(arena[((s * len(groups) + i) * 2) * words:((s * len(groups) + i) * 2 + 1) * words],
                   arena[((s * len(groups) + i) * 2 + 1) * words:((s * len(groups) + i) * 2 + 2) * words])
                  for i in range(len(groups))] for s in range(2)]
        pending = None
        ev = None
        if self.events is not None:
            import torch
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        for ci, row0 in enumerate(range(0, sub_rows, cr)):
            nrows = min(cr, sub_rows - row0)
            slot = slots[ci & 1]
            for (prank, ls, pat), (sbuf, _) in zip(groups, slot):
                self.local.pack(ls, pat, row0, nrows, sbuf)
            h = self.transport.start([sb for sb, _ in slot], [rb for _, rb in slot], [g[0] for g in groups],
                                     nrows * self.local.row_bytes)
            if pending is not None:
                self._drain(pending)
            pending = (h, groups, slot, row0, nrows)
            self.bytes_sent += nrows * self.local.row_bytes * len(groups)
            self.chunks += 1
        self._drain(pending)
        if ev is not None:
            ev[1].record()
            self.events.append(ev)

    def _drain(self, pending):
        h, groups, slot, row0, nrows = pending
        self.transport.finish(h)
        for (prank, ls, pat), (_, rbuf) in zip(groups, slot):
            self.local.unpack(ls, pat, row0, nrows, rbuf)


class TorchDistTransport:
    """Point-to-point transfers over torch.distributed (NCCL on GPUs, gloo in the CPU tests):
    all partners of a chunk in one batched group; finish() makes the current stream wait (NCCL)
    or blocks (gloo)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist

    def start(self, sends, recvs, peers, nbytes):
        ops = []
        for sb, rb, p in zip(sends, recvs, peers):
            n = nbytes // sb.element_size()
            ops.append(self.dist.P2POp(self.dist.isend, sb[:n], p))
            ops.append(self.dist.P2POp(self.dist.irecv, rb[:n], p))
        return self.dist.batch_isend_irecv(ops)

    def finish(self, works):
        for w in works:
            w.wait()


class DeviceShardLocal:
    """A shard = one libqbg register of the local qubits; pack / unpack are libqbg kernels into
    library-owned staging buffers (viewed as torch tensors for NCCL)."""

    def __init__(self, nl: int, seed: int = 42, dtype: str = "c128"):
        import torch
        from .register import Register
        self.torch = torch
        self.nl = nl
        self.reg = Register(nl, 1, seed, dtype)  # zero-filled by qbg_reg_create
        self.rows_per_shard = 1 << nl
        self.elem = 16 if dtype == "c128" else 8
        self.row_bytes = self.elem  # B = 1
        self._arena = None
        self.staging_high_water = 0

    def arena(self, nbytes):
        """The staging arena (library-owned device memory, grown only if a larger one is asked)."""
        import ctypes
        from ._capi import check, lib
        if self._arena is not None and self._arena[1] >= nbytes:
            return self._arena[2]
        self.release_staging()
        ptr = ctypes.c_void_p()
        check(lib().qbg_buffer_alloc(nbytes, ctypes.byref(ptr)))
        t = self.torch.as_tensor(_CudaBuf(ptr.value, nbytes // 8), device="cuda")
        self._arena = (ptr, nbytes, t)
        self.staging_high_water = max(self.staging_high_water, nbytes)
        return t

    def release_staging(self):
        from ._capi import lib
        if self._arena is not None:
            lib().qbg_buffer_free(self._arena[0])
            self._arena = None

    def _fix(self, ls):
        import ctypes
        arr = (ctypes.c_int32 * max(1, len(ls)))(*[l + 1 for l in ls])
        return arr, len(ls)

    def pack(self, ls, pat, row0, nrows, buf):
        from ._capi import check, lib
        arr, nf = self._fix(ls)
        check(lib().qbg_shard_pack(self.reg._h, arr, nf, pat, row0, nrows, buf.data_ptr()))

    def unpack(self, ls, pat, row0, nrows, buf):
        from ._capi import check, lib
        arr, nf = self._fix(ls)
        check(lib().qbg_shard_unpack(self.reg._h, arr, nf, pat, row0, nrows, buf.data_ptr()))

    def set_zero(self, amplitude_one: bool):
        from ._capi import check, lib
        if amplitude_one:
            check(lib().qbg_set_zero(self.reg._h))
        else:
            self.reg.scale(0.0)

    def apply(self, lops):
        apply_lops(self.reg, lops)

    def expect(self, terms) -> float:
        return expect_terms(self.reg, terms)

    def amplitudes(self) -> np.ndarray:
        return self.reg.state()[0]


class DistShardBackend:
    """One shard per rank; exchanges through `transport`.  The product configuration is
    DeviceNcclBackend (libqbg shard, NCCL); the CPU tests run this class with a gloo transport
    and a CPU shard, so the chunk loop, staging and transfers they check are this code."""

    def __init__(self, local, transport, rank: int, world: int, g: int, staging_bytes: int = DEFAULT_STAGING_BYTES,
                 allreduce=None):
        if world != 1 << g:
            raise errors.ValidationError("sharded: world size must be 2^g")
        self.local, self.rank, self.world, self.g = local, rank, world, g
        self.exchange = ChunkedExchange(local, transport, rank, staging_bytes)
        self._allreduce = allreduce
        self.set_zero()

    def set_zero(self):
        self.local.set_zero(self.rank == 0)

    def remap(self, pairs):
        self.exchange.remap(pairs)

    def apply_local(self, rank_ops):
        self.local.apply(rank_ops(self.rank))

    def expect_local(self, local_terms):
        return float(self.local.expect(local_terms(self.rank)))

    def reduce_sum(self, v: float) -> float:
        return self._allreduce(v) if self._allreduce else v

    def gather(self):
        import torch
        import torch.distributed as dist
        mine = torch.from_numpy(np.ascontiguousarray(self.local.amplitudes()).view(np.float64).copy())
        out = [torch.zeros_like(mine) for _ in range(self.world)]
        dist.all_gather(out, mine)
        return [o.numpy().view(np.complex128) for o in out]


def _nccl_allreduce(v: float) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


class DeviceNcclBackend(DistShardBackend):
    """One shard per process / GPU (libqbg register), exchanges with NCCL send/recv over NVLink
    through torch.distributed, staged in library-owned chunk buffers."""

    def __init__(self, n: int, g: int, seed: int = 42, dtype: str = "c128", staging_bytes: int = DEFAULT_STAGING_BYTES):
        import torch
        import torch.distributed as dist
        from ._capi import check, lib
        check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
        rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
        self.n, self.nl = n, n - g
        super().__init__(DeviceShardLocal(n - g, seed, dtype), TorchDistTransport(), rank, world, g, staging_bytes,
                         allreduce=_nccl_allreduce if world > 1 else None)

    def gather(self):
        import torch
        import torch.distributed as dist
        v = self.local.reg.state()[0]
        mine = torch.from_numpy(np.ascontiguousarray(v).view(np.float64).copy()).cuda()
        out = [torch.zeros_like(mine) for _ in range(self.world)]
        dist.all_gather(out, mine)
        return [o.cpu().numpy().view(np.complex128) for o in out]


class DeviceVirtualBackend:
    """All 2^g shards as libqbg registers on the current GPU; a remap runs the same chunked
    pack / unpack kernels, each rank unpacking straight from its partner's packed chunk."""

    def __init__(self, n: int, g: int, seed: int = 42, dtype: str = "c128", staging_bytes: int = DEFAULT_STAGING_BYTES):
        import torch
        from ._capi import check, lib
        check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
        self.n, self.g, self.nl = n, g, n - g
        self.locals = [DeviceShardLocal(self.nl, seed, dtype) for _ in range(1 << g)]
        self.staging_bytes = staging_bytes
        self.bytes_moved = 0
        self.set_zero()

    def set_zero(self):
        for r, lo in enumerate(self.locals):
            lo.set_zero(r == 0)

    def remap(self, pairs):
        if not pairs:
            return
        G = 1 << self.g
        sub_rows = (1 << self.nl) >> len(pairs)
        npart = (1 << len(pairs)) - 1
        per = self.staging_bytes // (G * npart)  # one packed chunk per (rank, partner)
        cr = max(1, per // self.locals[0].row_bytes)
        cr = min(sub_rows, 1 << (cr.bit_length() - 1))
        words = cr * self.locals[0].row_bytes // 8
        groups = [remap_groups(r, pairs) for r in range(G)]
        arenas = [lo.arena(npart * words * 8) for lo in self.locals]
        for row0 in range(0, sub_rows, cr):
            nrows = min(cr, sub_rows - row0)
            bufs = {}
            for r in range(G):
                for i, (prank, ls, pat) in enumerate(groups[r]):
                    b = arenas[r][i * words:(i + 1) * words]
                    self.locals[r].pack(ls, pat, row0, nrows, b)
                    bufs[(r, prank)] = b
            for r in range(G):  # each rank unpacks its partner's packed chunk in place
                for prank, ls, pat in groups[r]:
                    self.locals[r].unpack(ls, pat, row0, nrows, bufs[(prank, r)])
                    self.bytes_moved += nrows * self.locals[r].row_bytes

    def apply_local(self, rank_ops):
        for r, lo in enumerate(self.locals):
            lo.apply(rank_ops(r))

    def expect_local(self, local_terms):
        return sum(float(lo.expect(local_terms(r))) for r, lo in enumerate(self.locals))

    def reduce_sum(self, v: float) -> float:
        return v

    def gather(self):
        return [lo.amplitudes() for lo in self.locals]


# ---- helpers ----------------------------------------------------------------------------------------
class _CudaBuf:
    """__cuda_array_interface__ over a raw device pointer (float64 elements)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def _lops_key(nqubits, lops):
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    h.update(str(nqubits).encode())
    for o in lops:
        h.update(repr((o.kind, o.targets, o.ctrls, o.cfg)).encode())
        h.update(np.ascontiguousarray(o.mat, dtype=complex).tobytes())
        if o.perm is not None:
            h.update(np.ascontiguousarray(o.perm, dtype=np.int64).tobytes())
    return h.digest()


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


class _ProgCache:
    """Compiled segment programs by content (a repeated step re-uses its plans and kernels)."""

    def __init__(self, cap=512):
        from collections import OrderedDict
        self.d, self.cap = OrderedDict(), cap

    def get(self, nqubits, lops):
        from ._capi import lib
        k = _lops_key(nqubits, lops)
        h = self.d.get(k)
        if h is not None:
            self.d.move_to_end(k)
            return h
        h = lops_program(nqubits, lops)
        self.d[k] = h
        while len(self.d) > self.cap:
            _, old = self.d.popitem(last=False)
            lib().qbg_prog_destroy(old)
        return h


_PROGS = _ProgCache()


def apply_lops(reg, lops):
    """Applies realised local ops to a libqbg register as one fused program."""
    from ._capi import check, lib
    if not lops:
        return
    check(lib().qbg_apply(reg._h, _PROGS.get(reg.nqubits, lops)))


_OBS = {}


def expect_terms(reg, terms) -> float:
    """Re Σ c <ψ|P|ψ> for Pauli terms given as (c, xmask, zmask) over the register's qubits; the
    compiled observable (and its seed plans) is cached by content."""
    import ctypes
    from ._capi import QbgPauliTerm, check, lib
    if not terms:
        return 0.0
    key = (reg.nqubits, tuple((complex(c), int(x), int(z)) for c, x, z in terms))
    h = _OBS.get(key)
    if h is None:
        arr = (QbgPauliTerm * len(terms))()
        for k, (c, x, z) in enumerate(terms):
            arr[k] = QbgPauliTerm(complex(c).real, complex(c).imag, x, z)
        h = ctypes.c_void_p()
        check(lib().qbg_obs_create(reg.nqubits, arr, len(terms), ctypes.byref(h)))
        if len(_OBS) > 256:
            for old in _OBS.values():
                lib().qbg_obs_destroy(old)
            _OBS.clear()
        _OBS[key] = h
    out = np.empty(reg.nbatch)
    check(lib().qbg_expect(reg._h, h, out.ctypes.data))
    return float(out.sum())
