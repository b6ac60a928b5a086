"""Sharded state vectors (global qubits = rank bits, qubit-swap exchanges): the schedule and the
per-rank specialisation checked on CPU with numpy shards driven by the CPU oracle (single
process, and two gloo ranks exchanging halves through torch.distributed exactly like the NCCL
backend), and on one GPU with the virtual-rank device backend.  Reference: full-state oracle."""
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
from paper_1912_10877_b200.sharded import ShardedState, _half_view


def _mat(o):
    if o.kind == M.MAT_DIAGONAL:
        return M.Diagonal(o.mat)
    if o.kind == M.MAT_PERMUTATION:
        return M.Permutation(o.perm, o.mat)
    return M.Dense(o.mat)


class NumpyBackend:
    def __init__(self, n, g, orc):
        self.nl, self.g, self.orc = n - g, g, orc
        self.shards = [np.zeros((1, 1 << self.nl), complex) for _ in range(1 << g)]
        self.shards[0][0, 0] = 1

    def apply_local(self, rank_ops):
        for r in range(1 << self.g):
            for o in rank_ops(r):
                self.shards[r] = self.orc.instruct(self.shards[r], self.nl, _mat(o), [t + 1 for t in o.targets],
                                                   [c + 1 for c in o.ctrls], list(o.cfg))

    def _half(self, r, l, v):
        return self.shards[r].reshape(1 << (self.nl - l - 1), 2, 1 << l)[:, v]

    def swap(self, k, l):
        for r in range(1 << self.g):
            if (r >> k) & 1:
                continue
            p = r | (1 << k)
            a, b = self._half(r, l, 1), self._half(p, l, 0)
            tmp = a.copy()
            a[...] = b
            b[...] = tmp

    def expect_local(self, local_terms):
        return sum(float(self.orc.obs_apply(self.shards[r], local_terms(r))[1].sum()) for r in range(1 << self.g))

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
    np.testing.assert_allclose(st.state(), want, atol=1e-12)  # the expect swaps keep the state


class CpuDistBackend(NumpyBackend):
    """One shard per gloo rank; swap exactly as DeviceNcclBackend (pack half, sendrecv, unpack)."""

    def __init__(self, n, g, orc, rank):
        import torch.distributed as dist
        self.dist, self.rank = dist, rank
        self.nl, self.g, self.orc = n - g, g, orc
        self.shard = np.zeros((1, 1 << self.nl), complex)
        if rank == 0:
            self.shard[0, 0] = 1

    def apply_local(self, rank_ops):
        for o in rank_ops(self.rank):
            self.shard = self.orc.instruct(self.shard, self.nl, _mat(o), [t + 1 for t in o.targets],
                                           [c + 1 for c in o.ctrls], list(o.cfg))

    def swap(self, k, l):
        import torch
        b = (self.rank >> k) & 1
        part = self.rank ^ (1 << k)
        mine = self.shard.reshape(1 << (self.nl - l - 1), 2, 1 << l)[:, 1 - b]
        send = torch.from_numpy(np.ascontiguousarray(mine).view(np.float64).copy())
        recv = torch.empty_like(send)
        ops = [self.dist.P2POp(self.dist.isend, send, part), self.dist.P2POp(self.dist.irecv, recv, part)]
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()
        mine[...] = recv.numpy().view(np.complex128).reshape(mine.shape)

    def expect_local(self, local_terms):
        import torch
        e = torch.tensor([float(self.orc.obs_apply(self.shard, local_terms(self.rank))[1].sum())], dtype=torch.float64)
        self.dist.all_reduce(e)
        return float(e.item())

    def gather(self):
        import torch
        t = torch.from_numpy(self.shard[0].view(np.float64).copy())
        out = [torch.zeros_like(t) for _ in range(1 << self.g)]
        self.dist.all_gather(out, t)
        return [o.numpy().view(np.complex128) for o in out]


def _worker(rank, port, n, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    import oracle as O2
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(5).uniform(0, 2 * np.pi, B.nparameters(circ)))
    st = ShardedState(CpuDistBackend(n, 1, O2.restatement(), rank), n, 1).apply(circ)
    e = st.expect_pauli(B.pauli_terms(C.heisenberg(n)))
    out[rank] = (st.state(), e)
    dist.destroy_process_group()


def test_sharded_two_gloo_ranks(orc):
    n = 7
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(port, n, out), nprocs=2, join=True)
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(5).uniform(0, 2 * np.pi, B.nparameters(circ)))
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    _, e_ref = orc.obs_apply(want[None, :], B.pauli_terms(C.heisenberg(n)))
    for r in range(2):
        full, e = out[r]
        np.testing.assert_allclose(full, want, atol=1e-12)
        assert abs(e - e_ref[0]) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,g", [(14, 3), (16, 1)])
def test_sharded_virtual_device(orc, n, g):
    from paper_1912_10877_b200.sharded import DeviceVirtualBackend
    circ = _circuit(n)
    B.dispatch(circ, np.random.default_rng(n).uniform(0, 2 * np.pi, B.nparameters(circ)))
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    st = ShardedState(DeviceVirtualBackend(n, g), n, g).apply(circ)
    got = st.state()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
    terms = B.pauli_terms(C.heisenberg(n))
    _, e_ref = orc.obs_apply(want[None, :], terms)
    assert abs(st.expect_pauli(terms) - e_ref[0]) < 1e-12 * max(1, abs(e_ref[0])) * 10


@pytest.mark.parametrize("g,seed", [(1, 41), (2, 42), (3, 43)])
def test_sharded_random_circuits_numpy(orc, g, seed):
    """Every gate form (controls on global qubits, 2-qubit gates straddling the rank bits, dense
    4x4, diagonal gates on global qubits) through the swap schedule, vs the full-state oracle."""
    from test_gpu_random_circuits import random_circuit
    n = 9
    circ = random_circuit(n, 90, seed)
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    st = ShardedState(NumpyBackend(n, g, orc), n, g).apply(circ)
    got = st.state()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
    terms = B.pauli_terms(C.heisenberg(n))
    _, e_ref = orc.obs_apply(want[None, :], terms)
    assert abs(st.expect_pauli(terms) - e_ref[0]) < 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("n,g,seed", [(15, 3, 51), (17, 2, 52)])
def test_sharded_random_circuits_device(orc, n, g, seed):
    from paper_1912_10877_b200.sharded import DeviceVirtualBackend
    from test_gpu_random_circuits import random_circuit
    circ = random_circuit(n, 150, seed)
    want = orc.apply_program(O.Oracle.zero_state(n), n, _lowered(circ), B.parameters(circ))[0]
    st = ShardedState(DeviceVirtualBackend(n, g), n, g).apply(circ)
    got = st.state()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
