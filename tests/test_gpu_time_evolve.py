"""time_evolve (Listing 6): the device Lanczos exponential
vs the dense matrix exponential (oracle.expm_apply), and expect' through time-evolution nodes vs
central finite differences."""
import numpy as np
import pytest

import oracle as O
import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C
from paper_1912_10877_b200 import errors

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b))


def test_spec_example_heisenberg4(orc):
    """e^{-iHt}|ψ> = dense expm for heisenberg(4), t = 0.1, within 1e-8 (we hold 1e-12)."""
    n = 4
    h = C.heisenberg(n)
    st = orc.rand_state(n, 1, 7)
    want = O.expm_apply(st, B.pauli_terms(h), n, 0.1)
    reg = qb.Register(n, 1).set_state(st)
    qb.apply(reg, qb.time_evolve(h, 0.1))
    assert rel(reg.state(), want) < 1e-12


@pytest.mark.parametrize("n,nb,t", [(8, 1, 0.7), (10, 3, 2.5), (9, 2, -1.3)])
def test_vs_dense_expm(orc, n, nb, t):
    h = C.heisenberg(n, periodic=True)
    st = orc.rand_state(n, nb, n)
    want = O.expm_apply(st, B.pauli_terms(h), n, t)
    reg = qb.Register(n, nb).set_state(st)
    used = qb.evolve(reg, h, t)
    assert 1 <= used <= 30
    assert rel(reg.state(), want) < 1e-11


def test_identity_and_energy_conservation(orc):
    n = 12
    h = C.heisenberg(n)
    st = orc.rand_state(n, 1, 3)
    reg = qb.Register(n, 1).set_state(st)
    qb.apply(reg, qb.time_evolve(h, 0.0))
    assert np.array_equal(reg.state(), st)
    e0 = qb.expect(h, reg)[0]
    qb.apply(reg, qb.time_evolve(qb.cache(h), 1.7))  # Listing 6: time_evolve(cache(h), t)
    assert abs(qb.expect(h, reg)[0] - e0) < 1e-10 * max(1.0, abs(e0))
    assert abs(reg.norm(0) - 1.0) < 1e-12
    qb.apply(reg, B.dagger(qb.time_evolve(h, 1.7)))  # e^{+iHt} undoes it
    assert rel(reg.state(), st) < 1e-11


def test_circuit_with_time_evolution_grad_vs_fd(orc):
    n = 7
    h = C.heisenberg(n)
    te = qb.time_evolve(h, 0.37)
    circ = B.chain(n, C.variational_circuit(n, 1), te, B.put(n, 2, B.Rx(0.3)), B.put(n, (1, 5), B.rot(B.kron(B.Z, B.Z), 0.8)))
    B.dispatch(circ, np.random.default_rng(1).uniform(0, 2 * np.pi, B.nparameters(circ)))
    obs = qb.Add([B.put(n, 3, B.X), 0.5 * B.kron(n, ((1,), B.Z), ((4,), B.Y)), C.heisenberg(n)])
    st = orc.rand_state(n, 2, 5)
    reg = qb.Register(n, 2).set_state(st)
    res = qb.expect_grad(obs, (reg, circ), want_state_grad=True)
    th = B.parameters(circ)
    assert th.size == B.nparameters(circ) and any(nd is te for nd in B.parameter_nodes(circ))
    for k in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-5
        tm[k] -= 1e-5
        B.dispatch(circ, tp)
        ep = np.sum(qb.expect(obs, (reg, circ)))
        B.dispatch(circ, tm)
        em = np.sum(qb.expect(obs, (reg, circ)))
        assert abs((ep - em) / 2e-5 - res.param_grads[k]) < 1e-7, k
    B.dispatch(circ, th)
    np.testing.assert_allclose(res.energies, qb.expect(obs, (reg, circ)), atol=1e-12, rtol=0)


def test_errors():
    n = 4
    reg = qb.zero_state(n)
    with pytest.raises(errors.ValidationError):
        qb.apply(reg, qb.time_evolve(1j * B.put(n, 1, B.X), 0.2))  # non-hermitian
    with pytest.raises(errors.UnsupportedError):
        qb.time_evolve(B.put(20, 1, B.H), 0.2)  # not a Pauli expression and too large to materialise
    with pytest.raises(errors.UnsupportedError):
        qb.apply(reg, B.put(n, (1, 2), qb.time_evolve(C.heisenberg(2), 0.1)))


def _herm_block(n, seed):
    """A hermitian non-Pauli Hamiltonian: Σ of random hermitian 2-qubit matrices on random pairs."""
    rng = np.random.default_rng(seed)
    terms = []
    for _ in range(6):
        a, b = (int(v) for v in rng.choice(np.arange(1, n + 1), 2, replace=False))
        z = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
        terms.append(B.put(n, (a, b), B.matblock((z + z.conj().T) / 2)))
    return qb.Add(terms)


@pytest.mark.parametrize("n,nb", [(6, 1), (8, 3)])
def test_sparse_operator_apply_and_evolve(orc, n, nb):
    """The Cached / sparse path (matrix.hpp:680-724 matvec_cols): A|ψ> and e^{-iAt}|ψ>
    for a hermitian non-Pauli block vs dense numpy / expm."""
    import scipy.linalg
    h = _herm_block(n, n)
    A = B.mat(h)
    st = orc.rand_state(n, nb, 2)
    reg = qb.Register(n, nb).set_state(st)
    out = qb.sparse_operator(h).apply(reg)
    assert rel(out.state(), (A @ st.T).T) < 1e-13
    qb.apply(reg, qb.time_evolve(qb.cache(h), 0.6))
    want = (scipy.linalg.expm(-0.6j * A) @ st.T).T
    assert rel(reg.state(), want) < 1e-11


def test_sparse_time_evolution_grad_vs_fd():
    n = 6
    h = _herm_block(n, 3)
    circ = B.chain(n, C.variational_circuit(n, 1), qb.time_evolve(h, 0.45), B.put(n, 2, B.Ry(0.2)))
    B.dispatch(circ, np.random.default_rng(2).uniform(0, 2 * np.pi, B.nparameters(circ)))
    obs = C.heisenberg(n)
    reg = qb.zero_state(n)
    res = qb.expect_grad(obs, (reg, circ))
    th = B.parameters(circ)
    for k in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-5
        tm[k] -= 1e-5
        B.dispatch(circ, tp)
        ep = qb.expect(obs, (reg, circ))[0]
        B.dispatch(circ, tm)
        em = qb.expect(obs, (reg, circ))[0]
        assert abs((ep - em) / 2e-5 - res.param_grads[k]) < 1e-7, k
    B.dispatch(circ, th)


def test_sparse_errors():
    n = 4
    with pytest.raises(errors.ValidationError):  # non-hermitian
        qb.apply(qb.zero_state(n), qb.time_evolve(B.put(n, 1, B.S), 0.3))
