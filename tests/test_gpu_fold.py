"""Permutation folding: the CNOT / X gates at the start of a forward pass and at
the end of a checkpointed reverse pass are applied as an affine map of the tile's local index in
the load / store addressing.  CNOT networks with positive and negative controls, controls inside
and outside the tile, bare X gates and rotation runs between them, forward and expect' (the
checkpointed reverse pass with its TMA store) vs the CPU oracle at 1e-12 relative, complex128."""
import numpy as np
import pytest

import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C

from test_gpu_parity import lowered, rel

pytestmark = pytest.mark.gpu

TOL = 1e-12


def cnot_network(n, layers, seed):
    """Layers of a random CNOT chain (random direction and control value) and X gates, each
    followed by rotations on a random subset of the qubits."""
    rng = np.random.default_rng(seed)
    blocks = [B.put(n, q, B.Rx(float(rng.uniform(0, 6.28)))) for q in range(1, n + 1)]
    for _ in range(layers):
        order = rng.permutation(np.arange(1, n + 1))
        for i in range(n - 1):
            c, t = int(order[i]), int(order[i + 1])
            if rng.integers(0, 4) == 0:
                blocks.append(B.put(n, t, B.X))
            else:
                blocks.append(B.control(n, c if rng.integers(0, 3) else -c, t, B.X))
        for q in rng.choice(np.arange(1, n + 1), size=max(1, n // 2), replace=False):
            th = rng.uniform(0, 6.28, size=3)
            blocks.append(B.put(n, int(q), B.chain(B.Rz(float(th[0])), B.Rx(float(th[1])), B.Rz(float(th[2])))))
    return B.chain(n, *blocks)


def check(orc, circ, n, nb, seed):
    th = B.parameters(circ)
    em = lowered(circ)
    st = orc.rand_state(n, nb, seed)
    want = orc.apply_program(st, n, em, th)
    reg = qb.Register(n, nb).set_state(st)
    qb.apply(reg, circ)
    assert rel(reg.state(), want) < TOL
    h = C.heisenberg(n)
    e, g, _, sg = orc.expect_grad(st, n, em, th, B.pauli_terms(h))
    res = qb.expect_grad(h, (qb.Register(n, nb).set_state(st), circ), want_state_grad=True)
    assert np.abs(res.energies - e).max() <= TOL * max(1.0, np.abs(e).max())
    assert np.abs(res.param_grads - g).max() <= TOL * max(1.0, np.abs(g).max())
    assert rel(res.state_grad.state(), sg) < TOL


@pytest.mark.parametrize("n,layers,nb,seed", [(12, 6, 1, 1), (14, 5, 2, 2), (16, 4, 1, 3), (13, 6, 4, 4),
                                              (17, 3, 1, 5)])
def test_cnot_networks_vs_oracle(orc, n, layers, nb, seed):
    check(orc, cnot_network(n, layers, seed), n, nb, seed)


@pytest.mark.parametrize("n,d,seed", [(14, 4, 11), (18, 3, 12)])
def test_variational_ring_vs_oracle(orc, n, d, seed):
    """The bench's circuit family (CNOT ring incl. the wrap-around n -> 1 whose control lies outside
    most tiles), folded in both directions."""
    circ = C.variational_circuit(n, d)
    B.dispatch(circ, "random", rng=qb.Rng(seed))
    check(orc, circ, n, 1, seed)
