"""Randomised circuits over every gate form the planner lowers: single-qubit
constants and rotations, shift / phase, controlled gates with mixed control configurations,
2-qubit rotations (rot(XX), rot(ZZ)), SWAP / CZ / Toffoli, dense random 2x2 and 4x4 unitaries.
Forward and expect' through the fused JIT engine vs the CPU oracle (1e-12 relative, complex128)."""
import numpy as np
import pytest

import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C

from test_gpu_parity import lowered, rel

pytestmark = pytest.mark.gpu

TOL = 1e-12


def unitary(rng, d):
    z = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def random_circuit(n, ngates, seed):
    rng = np.random.default_rng(seed)
    blocks = []

    def locs(k):
        return tuple(int(v) for v in rng.choice(np.arange(1, n + 1), size=k, replace=False))

    for _ in range(ngates):
        kind = rng.integers(0, 12)
        th = float(rng.uniform(0, 2 * np.pi))
        if kind == 0:
            blocks.append(B.put(n, locs(1)[0], [B.X, B.Y, B.Z, B.H, B.T, B.S, B.Tdag][rng.integers(0, 7)]))
        elif kind == 1:
            blocks.append(B.put(n, locs(1)[0], [B.Rx, B.Ry, B.Rz][rng.integers(0, 3)](th)))
        elif kind == 2:
            blocks.append(B.put(n, locs(1)[0], B.shift(th)))
        elif kind == 3:
            blocks.append(B.put(n, locs(1)[0], B.phase(th)))
        elif kind == 4:
            t, c = locs(2)
            blocks.append(B.control(n, c if rng.integers(0, 2) else -c, t, [B.Rx, B.Ry, B.Rz][rng.integers(0, 3)](th)))
        elif kind == 5:
            t, c1, c2 = locs(3)
            blocks.append(B.control(n, (c1, -c2), t, B.X))
        elif kind == 6:
            a, b = locs(2)
            blocks.append(B.put(n, (a, b), B.rot(B.kron(B.X, B.X), th)))
        elif kind == 7:
            a, b = locs(2)
            blocks.append(B.put(n, (a, b), B.rot(B.kron(B.Z, B.Z), th)))
        elif kind == 8:
            a, b = locs(2)
            blocks.append(B.put(n, (a, b), [B.SWAP, B.CZ][rng.integers(0, 2)]))
        elif kind == 9:
            blocks.append(B.put(n, locs(1)[0], B.matblock(unitary(rng, 2))))
        elif kind == 10:
            a, b = locs(2)
            blocks.append(B.put(n, (a, b), B.matblock(unitary(rng, 4))))
        else:
            t, c = locs(2)
            blocks.append(B.control(n, c, t, B.shift(th)))
    return B.chain(n, *blocks)


def wide_circuit(n, ngates, seed):
    """Random circuits with 3-, 4- and 5-qubit blocks: dense unitaries, controlled dense blocks and
    rotations whose generators act on 3-5 qubits (forward and reverse through t <= 5)."""
    rng = np.random.default_rng(seed)
    blocks = []

    def locs(k):
        return tuple(int(v) for v in rng.choice(np.arange(1, n + 1), size=k, replace=False))

    paulis = [B.X, B.Y, B.Z]
    for _ in range(ngates):
        kind = rng.integers(0, 5)
        th = float(rng.uniform(0, 2 * np.pi))
        t = int(rng.integers(3, 6))
        if kind == 0:
            blocks.append(B.put(n, locs(t), B.matblock(unitary(rng, 1 << t))))
        elif kind == 1:
            q = locs(t + 1)
            blocks.append(B.control(n, q[t], q[:t], B.matblock(unitary(rng, 1 << t))))
        elif kind == 2:
            gen = B.kron(*[paulis[int(rng.integers(0, 3))] for _ in range(t)])
            blocks.append(B.put(n, locs(t), B.rot(gen, th)))
        elif kind == 3:
            q = locs(t + 1)
            gen = B.kron(*[paulis[int(rng.integers(0, 3))] for _ in range(t)])
            blocks.append(B.control(n, -q[t], q[:t], B.rot(gen, th)))
        else:
            blocks.append(B.put(n, locs(1)[0], [B.Rx, B.Ry, B.Rz][rng.integers(0, 3)](th)))
    return B.chain(n, *blocks)


@pytest.mark.parametrize("n,ngates,nb,seed", [(7, 30, 1, 71), (12, 40, 2, 72), (16, 30, 1, 73)])
def test_wide_gates_forward_and_grad(orc, n, ngates, nb, seed):
    """expect' through 3-5-qubit gates (reverse mode with t <= 5 and 5-qubit generators) vs the oracle."""
    circ = wide_circuit(n, ngates, seed)
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


CASES = [(5, 60, 1, 1), (9, 120, 2, 2), (12, 150, 1, 3), (14, 200, 4, 4), (20, 250, 1, 5), (22, 160, 1, 6)] + \
    [(n, 120, nb, 10 + s) for s, (n, nb) in enumerate([(12, 1), (13, 2), (14, 1), (15, 3), (16, 1), (16, 8),
                                                      (17, 1), (12, 32), (11, 1), (11, 4), (13, 6)])]


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "pergate"])
@pytest.mark.parametrize("n,ngates,nb,seed", CASES)
def test_random_circuit_forward_and_grad(orc, fused, n, ngates, nb, seed):
    if not fused and n >= 20:
        pytest.skip("per-gate path covered at the smaller sizes")
    qb.set_fusion(fused)
    try:
        circ = random_circuit(n, ngates, seed)
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
        # energies / gradients relative to the observable scale (|E| can be ~1e-3 of ||O||)
        assert np.abs(res.energies - e).max() <= TOL * max(1.0, np.abs(e).max())
        assert np.abs(res.param_grads - g).max() <= TOL * max(1.0, np.abs(g).max())
        assert rel(res.state_grad.state(), sg) < TOL
    finally:
        qb.set_fusion(True)


@pytest.mark.parametrize("n,seed", [(12, 21), (14, 22)])
def test_random_circuit_c64(orc, n, seed):
    """complex64 through the same fused kernels: within 1e-5 of the complex128 oracle."""
    circ = random_circuit(n, 120, seed)
    th = B.parameters(circ)
    em = lowered(circ)
    st = orc.rand_state(n, 1, seed)
    want = orc.apply_program(st, n, em, th)
    reg = qb.Register(n, 1, dtype="c64").set_state(st)
    qb.apply(reg, circ)
    assert rel(reg.state(), want) < 1e-5
    h = C.heisenberg(n)
    e, g, _, _ = orc.expect_grad(st, n, em, th, B.pauli_terms(h))
    res = qb.expect_grad(h, (qb.Register(n, 1, dtype="c64").set_state(st), circ))
    assert np.abs(res.energies - e).max() < 1e-5 * max(1.0, np.abs(e).max())
    assert np.abs(res.param_grads - g).max() < 1e-5 * max(1.0, np.abs(g).max())


def random_observable(n, nterms, seed):
    """Σ c_t P_t with random real weights on random Pauli strings (1-4 non-identity factors)."""
    rng = np.random.default_rng(seed)
    terms = []
    for _ in range(nterms):
        k = int(rng.integers(1, 5))
        qs = rng.choice(np.arange(1, n + 1), size=k, replace=False)
        ps = [[B.X, B.Y, B.Z][int(rng.integers(0, 3))] for _ in range(k)]
        terms.append(float(rng.normal()) * B.kron(n, *[((int(q),), p) for q, p in zip(qs, ps)]))
    return qb.Add(terms)


@pytest.mark.parametrize("n,nb,seed", [(12, 1, 31), (15, 2, 32), (18, 1, 33)])
def test_random_observable_expect_and_grad(orc, n, nb, seed):
    """The seed planner (Pauli groups by X support, Y phases, Z masks inside / outside the tile)."""
    circ = random_circuit(n, 80, seed)
    th = B.parameters(circ)
    em = lowered(circ)
    obs = random_observable(n, 25, seed)
    st = orc.rand_state(n, nb, seed)
    e, g, _, sg = orc.expect_grad(st, n, em, th, B.pauli_terms(obs))
    res = qb.expect_grad(obs, (qb.Register(n, nb).set_state(st), circ), want_state_grad=True)
    assert np.abs(res.energies - e).max() <= TOL * max(1.0, np.abs(e).max())
    assert np.abs(res.param_grads - g).max() <= TOL * max(1.0, np.abs(g).max())
    assert rel(res.state_grad.state(), sg) < TOL
    ex = qb.expect(obs, (qb.Register(n, nb).set_state(st), circ))
    assert np.abs(ex - e).max() <= TOL * max(1.0, np.abs(e).max())
