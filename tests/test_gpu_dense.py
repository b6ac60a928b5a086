"""Dense 3..5-qubit blocks on the FP64 tensor cores (dense_mma.cu, DMMA m8n8k4) and gate fusion
into dense k-qubit blocks (densefuse.py, BASELINE cfg 4), vs the CPU oracle (1e-12)."""
import numpy as np
import pytest

import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200.densefuse import fuse_dense

from test_gpu_parity import lowered, rel
from test_gpu_random_circuits import unitary

pytestmark = pytest.mark.gpu


@pytest.fixture
def per_gate():
    qb.set_fusion(False)  # every dense 3..5-qubit gate is its own launch of the DMMA kernel
    yield
    qb.set_fusion(True)


@pytest.mark.parametrize("n,nb", [(9, 1), (12, 2), (16, 1), (10, 4)])
def test_dense_blocks_every_placement(orc, per_gate, n, nb):
    rng = np.random.default_rng(n * 10 + nb)
    blocks = []
    for t in (3, 4, 5):
        for locs in [tuple(range(1, t + 1)), tuple(range(n - t + 1, n + 1)),
                     tuple(int(v) for v in rng.choice(np.arange(1, n + 1), size=t, replace=False))]:
            blocks.append(B.put(n, locs, B.matblock(unitary(rng, 1 << t))))
        q = [int(v) for v in rng.choice(np.arange(1, n + 1), size=t + 2, replace=False)]
        blocks.append(B.control(n, (q[t], -q[t + 1]), tuple(q[:t]), B.matblock(unitary(rng, 1 << t))))
    circ = B.chain(n, *blocks)
    st = orc.rand_state(n, nb, n)
    want = orc.apply_program(st, n, lowered(circ), B.parameters(circ))
    reg = qb.Register(n, nb).set_state(st)
    qb.apply(reg, circ)
    assert rel(reg.state(), want) < 1e-12


@pytest.mark.parametrize("n,d,k", [(12, 3, 5), (14, 2, 4), (13, 2, 3)])
def test_fuse_dense_variational(orc, per_gate, n, d, k):
    circ = qb.variational_circuit(n, d)
    qb.dispatch(circ, "random", rng=qb.Rng(n))
    fused = fuse_dense(circ, k)
    assert all(len(b.locs) <= k for b in fused.blocks)
    want = orc.apply_program(orc.zero_state(n), n, lowered(circ), B.parameters(circ))
    reg = qb.zero_state(n)
    qb.apply(reg, fused)
    assert rel(reg.state(), want) < 1e-12


@pytest.mark.parametrize("n,nb", [(11, 1), (13, 2), (12, 4)])
@pytest.mark.parametrize("path", ["tf32-tensor", "fp64-tensor", "cuda"])
def test_dense_blocks_c64_paths(orc, per_gate, n, nb, path):
    """complex64 dense 3..5-qubit blocks through every dense path — tcgen05 (kind::tf32, 3-piece
    split), the FP64 tensor cores (widened), the CUDA cores — within 1e-5 of the complex128 oracle
    (plain TF32 would be ~1e-3)."""
    qb.set_dense_path(path)
    rng = np.random.default_rng(n * 7 + nb)
    blocks = []
    for t in (3, 4, 5):
        for locs in [tuple(range(1, t + 1)), tuple(range(n - t + 1, n + 1)),
                     tuple(int(v) for v in rng.choice(np.arange(1, n + 1), size=t, replace=False))]:
            blocks.append(B.put(n, locs, B.matblock(unitary(rng, 1 << t))))
        q = [int(v) for v in rng.choice(np.arange(1, n + 1), size=t + 2, replace=False)]
        blocks.append(B.control(n, (q[t], -q[t + 1]), tuple(q[:t]), B.matblock(unitary(rng, 1 << t))))
    circ = B.chain(n, *blocks)
    st = orc.rand_state(n, nb, n)
    want = orc.apply_program(st, n, lowered(circ), B.parameters(circ))
    try:
        reg = qb.Register(n, nb, dtype="c64").set_state(st)
        qb.apply(reg, circ)
    finally:
        qb.set_dense_path("fp64-tensor")
    assert rel(reg.state(), want) < 1e-5


def test_fuse_dense_variational_c64(orc, per_gate):
    n = 14
    circ = qb.variational_circuit(n, 3)
    qb.dispatch(circ, "random", rng=qb.Rng(3))
    want = orc.apply_program(orc.zero_state(n), n, lowered(circ), B.parameters(circ))
    reg = qb.zero_state(n, dtype="c64")
    qb.apply(reg, fuse_dense(circ, 5))
    assert rel(reg.state(), want) < 1e-5


@pytest.mark.parametrize("n,nb,dtype", [(14, 1, "c128"), (13, 2, "c128"), (12, 1, "c64")])
@pytest.mark.parametrize("t", [3, 4])
def test_dense_blocks_fused_in_tiles(orc, n, nb, dtype, t):
    """3- and 4-qubit dense gates (matblocks, with and without controls) are stage ops of the tile
    passes (OP_DENSE3 / OP_DENSE4): forward and expect' (rotations between them) vs the oracle."""
    rng = np.random.default_rng(n + nb + t)
    blocks = []
    for layer in range(3):
        for s in range(0, n - t + 1, t):
            q = tuple(int(v) for v in rng.permutation(np.arange(1, n + 1))[:t])
            blocks.append(B.put(n, q, B.matblock(unitary(rng, 1 << t))))
        c = [int(v) for v in rng.permutation(np.arange(1, n + 1))[:t + 1]]
        blocks.append(B.control(n, c[t], tuple(c[:t]), B.matblock(unitary(rng, 1 << t))))
        for q in range(1, n + 1):
            blocks.append(B.put(n, q, [B.Rx, B.Ry, B.Rz][int(rng.integers(0, 3))](float(rng.uniform(0, 6.28)))))
    circ = B.chain(n, *blocks)
    plan = qb.compile_block(circ).plan_preview(nb, dtype)
    assert "single gate" not in plan.split("plan dir=2")[0]  # every forward gate tiled
    st = orc.rand_state(n, nb, n)
    want = orc.apply_program(st, n, lowered(circ), B.parameters(circ))
    tol = 1e-12 if dtype == "c128" else 1e-5
    reg = qb.Register(n, nb, dtype=dtype).set_state(st)
    qb.apply(reg, circ)
    assert rel(reg.state(), want) < tol
    h = qb.heisenberg(n)
    e, g, _, _ = orc.expect_grad(st, n, lowered(circ), B.parameters(circ), B.pauli_terms(h))
    res = qb.expect_grad(h, (qb.Register(n, nb, dtype=dtype).set_state(st), circ))
    assert np.abs(res.energies - e).max() <= tol * max(1.0, np.abs(e).max())
    assert np.abs(res.param_grads - g).max() <= tol * max(1.0, np.abs(g).max())
