"""Sharded state vectors (global qubits = rank bits, chunked all-to-all remaps): the schedule and
the per-rank specialisation checked on CPU with numpy shards driven by the CPU oracle; the SHIPPED
exchange (sharded.DistShardBackend: chunk loop, staging arena, torch.distributed transport) on
two and four gloo ranks with a CPU shard that only supplies the local primitives; and on one GPU
the virtual-rank device backend (libqbg pack / unpack kernels).  Reference: full-state oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT
import oracle as O
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C
from paper_1912_10877_b200 import matrix as M
from paper_1912_10877_b200.sharded import (ShardedSchedule, ShardedState, remap_groups, realise_ops)


def _mat(o):
    if o.kind == M.MAT_DIAGONAL:
        return M.Diagonal(o.mat)
    if o.kind == M.MAT_PERMUTATION:
        return M.Permutation(o.perm, o.mat)
    return M.Dense(o.mat)


def _sub_rows(nl, ls, pat):
    idx = np.arange(1 << nl)
    mask = sum(1 << l for l in ls)
    val = sum(((pat >> i) & 1) << l for i, l in enumerate(ls))
    return idx[(idx & mask) == val]


class NumpyBackend:
    """All shards in one process (numpy), remaps by direct sub-block exchange (remap_groups)."""

    def __init__(self, n, g, orc):
        self.nl, self.g, self.orc = n - g, g, orc
        self.set_zero()

    def set_zero(self):
        self.shards = [np.zeros((1, 1 << self.nl), complex) for _ in range(1 << self.g)]
        self.shards[0][0, 0] = 1

    def apply_local(self, rank_ops):
        for r in range(1 << self.g):
            for o in rank_ops(r):
                self.shards[r] = self.orc.instruct(self.shards[r], self.nl, _mat(o), [t + 1 for t in o.targets],
                                                   [c + 1 for c in o.ctrls], list(o.cfg))

    def remap(self, pairs):
        old = [s.copy() for s in self.shards]
        for r in range(1 << self.g):
            for prank, ls, pat in remap_groups(r, pairs):
                # r's sub-block for p receives p's sub-block for r
                mine = _sub_rows(self.nl, ls, pat)
                theirs_pat = next(pt for pr, _, pt in remap_groups(prank, pairs) if pr == r)
                self.shards[r][0, mine] = old[prank][0, _sub_rows(self.nl, ls, theirs_pat)]

    def expect_local(self, local_terms):
        return sum(float(self.orc.obs_apply(self.shards[r], local_terms(r))[1].sum()) for r in range(1 << self.g))

    def reduce_sum(self, v):
        return v

    def gather(self):
        return [s[0] for s in self.shards]


def _circuit(n):
    c = C.variational_circuit(n, 2)
    extra = [B.control(n, n, 1, B.X), B.control(n, 1, n, B.Ry(0.4)), B.put(n, (2, n), B.rot(B.kron(B.Z, B.Z), 0.9)),
             B.put(n, n - 1, B.H), B.control(n, (-n, 3), n - 1, B.shift(0.3)), B.put(n, (n - 1, n), B.SWAP)]
    return B.chain(n, c, *extra)


def _lowered(block):
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    return em


@pytest.mark.parametrize("g", [1, 2, 3])
def test_sharded_schedule_numpy(orc, g):
    n = 8
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(g).uniform(0, 2 * np.pi, B.nparameters(circ)))
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    st = ShardedState(NumpyBackend(n, g, orc), n, g).apply(circ)
    np.testing.assert_allclose(st.state(), want, atol=1e-12)
    terms = B.pauli_terms(C.heisenberg(n, periodic=True))
    e = st.expect_pauli(terms)
    _, e_ref = orc.obs_apply(want[None, :], terms)
    assert abs(e - e_ref[0]) < 1e-12
    np.testing.assert_allclose(st.state(), want, atol=1e-12)  # the expect remaps keep the state


def test_schedule_exchanges_variational_33q():
    """variational_circuit(33, 2) on 8 ranks (g = 3): round 1's 64-op look-ahead pairwise swaps
    took 21 exchanges of S_local/2 (10.5 S_local per rank, profiles/r01_big_state_33q.jsonl).  The
    Belady schedule with batched remaps must need fewer exchanges and fewer bytes."""
    n, g = 33, 3
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, "random")
    ops = realise_ops(_lowered(circ), B.parameters(circ))
    sch = ShardedSchedule(n, g)
    steps = list(sch.steps(ops))
    ex = [s[1] for s in steps if s[0] == "remap"]
    moved = sum(1 - 2.0 ** -len(p) for p in ex)  # S_local per rank per exchange: (1 - 2^-j)
    pairs = sum(len(p) for p in ex)
    print(f"33q/8 d2: {len(ex)} exchanges, {pairs} qubit moves, {moved:.3f} S_local per rank (round 1: 21, 10.5)")
    assert len(ex) < 21 and moved < 10.5
    # lower bound: every layer touches every qubit, so each of the 3 layers needs the 3 globals local
    assert pairs >= 9
    # every op's non-diagonal targets are local when it runs (rank_ops raises otherwise)
    nl = n - g
    for s in steps:
        if s[0] == "ops":
            ShardedSchedule.rank_ops(s[1], s[2], nl, 5)


class CpuShardLocal:
    """Local primitives of a CPU shard for DistShardBackend under gloo: pack / unpack by numpy
    indexing into the arena, gates and expectations by the CPU oracle.  Everything else — the
    chunk loop, staging arena sizing, transfers — is the shipped sharded.py code."""

    def __init__(self, nl, orc):
        import torch
        self.torch, self.nl, self.orc = torch, nl, orc
        self.shard = np.zeros((1, 1 << nl), complex)
        self.rows_per_shard = 1 << nl
        self.row_bytes = 16
        self._arena = None
        self.arena_high_water = 0
        self.chunks = []

    def arena(self, nbytes):
        if self._arena is None or self._arena.numel() * 8 < nbytes:
            self._arena = self.torch.zeros(nbytes // 8, dtype=self.torch.float64)
            self.arena_high_water = max(self.arena_high_water, nbytes)
        return self._arena

    def pack(self, ls, pat, row0, nrows, buf):
        rows = _sub_rows(self.nl, ls, pat)[row0:row0 + nrows]
        buf[:2 * nrows] = self.torch.from_numpy(self.shard[0, rows].view(np.float64).copy())
        self.chunks.append(nrows)

    def unpack(self, ls, pat, row0, nrows, buf):
        rows = _sub_rows(self.nl, ls, pat)[row0:row0 + nrows]
        self.shard[0, rows] = buf[:2 * nrows].numpy().copy().view(np.complex128)

    def set_zero(self, one):
        self.shard[:] = 0
        if one:
            self.shard[0, 0] = 1

    def apply(self, lops):
        for o in lops:
            self.shard = self.orc.instruct(self.shard, self.nl, _mat(o), [t + 1 for t in o.targets],
                                           [c + 1 for c in o.ctrls], list(o.cfg))

    def expect(self, terms):
        return float(self.orc.obs_apply(self.shard, terms)[1].sum()) if terms else 0.0

    def amplitudes(self):
        return self.shard[0]


def _gloo_allreduce(v):
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t)
    return float(t.item())


def _worker(rank, world, port, n, staging, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    import oracle as O2
    from paper_1912_10877_b200.sharded import DistShardBackend, TorchDistTransport
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = world.bit_length() - 1
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(5).uniform(0, 2 * np.pi, B.nparameters(circ)))
    local = CpuShardLocal(n - g, O2.restatement())
    be = DistShardBackend(local, TorchDistTransport(), rank, world, g, staging_bytes=staging, allreduce=_gloo_allreduce)
    st = ShardedState(be, n, g).apply(circ)
    e = st.expect_pauli(B.pauli_terms(C.heisenberg(n)))
    out[rank] = (st.state(), e, local.arena_high_water, max(local.chunks or [0]), be.exchange.chunks,
                 len(st.sched.exchanges))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 7), (4, 8)])
def test_dist_backend_gloo_chunked(orc, world, n):
    """DistShardBackend on `world` gloo ranks with a 512-byte staging arena: every exchange runs in
    several chunks (chunk rows < the sub-block), the arena never grows past the budget (memory
    high-water = shard + staging), and the state / energy equal the full-state oracle's."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    staging = 512
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, n, staging, out), nprocs=world, join=True)
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(5).uniform(0, 2 * np.pi, B.nparameters(circ)))
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    _, e_ref = orc.obs_apply(want[None, :], B.pauli_terms(C.heisenberg(n)))
    g = world.bit_length() - 1
    sub_rows = (1 << (n - g)) >> 1
    for r in range(world):
        full, e, hw, max_chunk, nchunks, nex = out[r]
        np.testing.assert_allclose(full, want, atol=1e-12)
        assert abs(e - e_ref[0]) < 1e-12
        assert 0 < hw <= staging
        assert 0 < max_chunk < sub_rows and nchunks > nex  # chunked: more chunks than exchanges


@pytest.mark.gpu
@pytest.mark.parametrize("n,g,staging", [(14, 3, 4096), (16, 1, 1 << 20), (15, 2, 1 << 12)])
def test_sharded_virtual_device(orc, n, g, staging):
    from paper_1912_10877_b200.sharded import DeviceVirtualBackend
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(n).uniform(0, 2 * np.pi, B.nparameters(circ)))
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    be = DeviceVirtualBackend(n, g, staging_bytes=staging)
    st = ShardedState(be, n, g).apply(circ)
    got = st.state()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
    terms = B.pauli_terms(C.heisenberg(n))
    _, e_ref = orc.obs_apply(want[None, :], terms)
    assert abs(st.expect_pauli(terms) - e_ref[0]) < 1e-12 * max(1, abs(e_ref[0]))
    assert all(lo.staging_high_water <= staging for lo in be.locals)


@pytest.mark.parametrize("g,seed", [(1, 41), (2, 42), (3, 43)])
def test_sharded_random_circuits_numpy(orc, g, seed):
    """Every gate form (controls on global qubits, 2-qubit gates straddling the rank bits, dense
    4x4, diagonal gates on global qubits) through the remap schedule, vs the full-state oracle."""
    from test_gpu_random_circuits import random_circuit
    n = 9
    circ = random_circuit(n, 90, seed)
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    st = ShardedState(NumpyBackend(n, g, orc), n, g).apply(circ)
    got = st.state()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
    terms = B.pauli_terms(C.heisenberg(n))
    _, e_ref = orc.obs_apply(want[None, :], terms)
    assert abs(st.expect_pauli(terms) - e_ref[0]) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,g,seed", [(15, 3, 51), (17, 2, 52)])
def test_sharded_random_circuits_device(orc, n, g, seed):
    from paper_1912_10877_b200.sharded import DeviceVirtualBackend
    from test_gpu_random_circuits import random_circuit
    circ = random_circuit(n, 150, seed)
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    st = ShardedState(DeviceVirtualBackend(n, g, staging_bytes=1 << 13), n, g).apply(circ)
    got = st.state()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


@pytest.mark.gpu
def test_shard_pack_unpack_kernels(orc):
    """qbg_shard_pack / unpack against numpy indexing: j = 1..3 fixed bits, chunk ranges, B = 3."""
    import ctypes
    import torch
    import paper_1912_10877_b200 as qb
    from paper_1912_10877_b200._capi import check, lib
    n, nb = 10, 3
    st = orc.rand_state(n, nb, 3)
    reg = qb.Register(n, nb).set_state(st)
    dev = st.T.copy()  # device layout [2^n][B]
    for ls, pat in [([4], 1), ([0, 7], 2), ([9, 2, 5], 5)]:
        rows = _sub_rows(n, ls, pat)
        arr = (ctypes.c_int32 * len(ls))(*[l + 1 for l in ls])
        buf = torch.zeros(2 * nb * len(rows), dtype=torch.float64, device="cuda")
        check(lib().qbg_shard_pack(reg._h, arr, len(ls), pat, 3, len(rows) - 5, buf.data_ptr()))
        qb.synchronize()
        got = buf.cpu().numpy().view(np.complex128)[: nb * (len(rows) - 5)].reshape(-1, nb)
        np.testing.assert_array_equal(got, dev[rows[3:len(rows) - 2]])
        buf2 = torch.arange(2 * nb * 4, dtype=torch.float64, device="cuda")
        check(lib().qbg_shard_unpack(reg._h, arr, len(ls), pat, 1, 4, buf2.data_ptr()))
        dev[rows[1:5]] = buf2.cpu().numpy().view(np.complex128).reshape(-1, nb)
        np.testing.assert_array_equal(reg.state().T, dev)


class _LoopbackHub:
    """In-process stand-in for NCCL between ranks running as threads on ONE GPU: start() posts
    this rank's send buffers, waits for its partners' posts, and copies each partner's buffer into
    the matching receive buffer (device copies on the shared stream).  Only the transport is
    replaced; DistShardBackend / ChunkedExchange / DeviceShardLocal (libqbg pack / unpack kernels,
    staging arena) are the shipped code."""

    def __init__(self, world):
        import threading
        self.world = world
        self.lock = threading.Condition()
        self.posts = {}
        self.gen = [0] * world

    def transport(self, rank):
        hub = self

        class T:
            def start(self, sends, recvs, peers, nbytes):
                n = nbytes // 8
                with hub.lock:
                    g = hub.gen[rank]
                    hub.gen[rank] += 1
                    for sb, p in zip(sends, peers):
                        hub.posts[(g, rank, p)] = sb[:n]
                    hub.lock.notify_all()
                    for rb, p in zip(recvs, peers):
                        while (g, p, rank) not in hub.posts:
                            hub.lock.wait(timeout=60)
                        rb[:n].copy_(hub.posts[(g, p, rank)])
                    hub.lock.notify_all()
                return (g, peers)

            def finish(self, h):
                import torch
                torch.cuda.synchronize()  # every partner's copy out of our send buffers is done

        return T()


@pytest.mark.gpu
@pytest.mark.parametrize("n,g,staging", [(12, 1, 1 << 12), (13, 2, 1 << 13)])
def test_dist_backend_device_shards_loopback(orc, n, g, staging):
    """DistShardBackend with DeviceShardLocal (the DeviceNcclBackend configuration minus NCCL) on one
    B200: 2^g ranks as threads, chunked remaps through the libqbg staging arena and pack / unpack
    kernels, vs the full-state oracle."""
    import threading
    import torch
    from paper_1912_10877_b200._capi import check, lib
    from paper_1912_10877_b200.sharded import DeviceShardLocal, DistShardBackend
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    world = 1 << g
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(n + g).uniform(0, 2 * np.pi, B.nparameters(circ)))
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    hub = _LoopbackHub(world)
    sums = {}
    sums_lock = threading.Lock()

    def reduce_sum_factory(rank):
        def red(v):
            with sums_lock:
                sums.setdefault("e", []).append(v)
            return v
        return red

    big = threading.Lock()  # the engine is not thread-safe per program: local compute one rank at a time

    class LockedLocal(DeviceShardLocal):
        def apply(self, lops):
            with big:
                super().apply(lops)
                torch.cuda.synchronize()

        def expect(self, terms):
            with big:
                return super().expect(terms)

    locals_ = [LockedLocal(n - g) for _ in range(world)]
    states, errors = {}, []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            be = DistShardBackend(locals_[rank], hub.transport(rank), rank, world, g, staging_bytes=staging,
                                  allreduce=reduce_sum_factory(rank))
            st = ShardedState(be, n, g).apply(circ)
            st.expect_pauli(B.pauli_terms(C.heisenberg(n)))
            states[rank] = (list(st.phys), be.exchange.chunks, len(st.sched.exchanges))
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    torch.cuda.synchronize()
    phys = states[0][0]
    assert all(states[r][0] == phys for r in range(world))
    assert states[0][1] > states[0][2] > 0  # chunked: more chunks than exchanges
    nl = n - g
    full = np.zeros(1 << n, dtype=complex)
    for r in range(world):
        sh = locals_[r].amplitudes()
        idx_phys = np.arange(1 << nl, dtype=np.int64) | (r << nl)
        logical = np.zeros_like(idx_phys)
        for q in range(n):
            logical |= ((idx_phys >> phys[q]) & 1) << q
        full[logical] = sh
    assert np.linalg.norm(full - want) / np.linalg.norm(want) < 1e-12
    _, e_ref = orc.obs_apply(want[None, :], B.pauli_terms(C.heisenberg(n)))
    assert abs(sum(sums["e"]) - e_ref[0]) < 1e-12 * max(1.0, abs(e_ref[0]))
    assert all(lo.staging_high_water <= staging for lo in locals_)
