"""Batch-sharded reverse-AD over torch.distributed (gloo, world size 2, CPU): the collective
logic of paper_1912_10877_b200.dist with the CPU oracle as the per-rank step, compared with the
single-process full-batch gradient.  CPU only."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lowered(block):
    from paper_1912_10877_b200 import blocks as B
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    return em


def _problem(n, nbatch):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_1912_10877_b200 import blocks as B
    from paper_1912_10877_b200 import circuits as C
    from paper_1912_10877_b200 import dist as D
    orc = O.restatement()
    circ = C.variational_circuit(n, 2)
    th = orc.dispatch_random(B.nparameters(circ), 42)
    B.dispatch(circ, th)
    bits = D.product_batch(n, nbatch, 42)
    st = np.zeros((nbatch, 1 << n), dtype=np.complex128)
    st[np.arange(nbatch), bits] = 1
    return orc, circ, th, st, B.pauli_terms(C.heisenberg(n))


def _worker(rank, world, port, n, nbatch, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_1912_10877_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, circ, th, st, terms = _problem(n, nbatch)
    lo, hi = D.shard_range(nbatch, rank, world)
    em = _lowered(circ)

    def step(obs, circuit, local):
        e, g, _, _ = orc.expect_grad(local, n, em, th, terms)
        return e, g

    e, g = D.sharded_expect_grad(None, circ, st[lo:hi], nbatch, local_step=step)
    out[rank] = (e, g)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nbatch", [6, 7])
def test_sharded_grad_equals_full_batch(nbatch):
    n = 5
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, n, nbatch, out), nprocs=2, join=True)
    orc, circ, th, st, terms = _problem(n, nbatch)
    e_full, g_full, _, _ = orc.expect_grad(st, n, _lowered(circ), th, terms)
    for r in range(2):
        e, g = out[r]
        np.testing.assert_allclose(e, e_full, atol=1e-13, rtol=0)
        np.testing.assert_allclose(g, g_full, atol=1e-12, rtol=0)


def test_shard_range_partitions():
    from paper_1912_10877_b200.dist import shard_range
    for B in (1, 7, 1000):
        for w in (1, 2, 3, 8):
            rs = [shard_range(B, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
