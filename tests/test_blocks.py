"""Host-side block logic: parameters order, dispatch, gatecount goldens,
Pauli expansion of observables, and the lowering semantics (lowered program == dense block
operator) checked through the CPU oracle.  CPU only."""
import numpy as np
import pytest

import oracle as O
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C
from paper_1912_10877_b200 import errors


def lowered(block):
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    return em


def test_gatecount_listing9_golden():
    """PAPER.md:580-588 / SPEC.md:767: variational_circuit(10, 10000)."""
    c = C.variational_circuit(10, 10000)
    gc = B.gatecount(c)
    assert gc == {"Rx": 100010, "Rz": 200000, "Control{X}": 100000}
    assert B.nparameters(c) == 300010


def test_variational_structure_counts():
    for n, d in [(25, 10), (20, 10), (4, 3)]:
        c = C.variational_circuit(n, d)
        assert len(lowered(c).ops) == n * (1 + 4 * d)
        assert B.nparameters(c) == n * (1 + 3 * d)


def test_parameters_dispatch_roundtrip_and_shared_nodes():
    c = C.variational_circuit(3, 2)
    v = np.arange(B.nparameters(c), dtype=float) / 7
    B.dispatch(c, v)
    assert np.array_equal(B.parameters(c), v)
    B.dispatch(c, lambda a, b: a - b, np.ones_like(v))
    np.testing.assert_allclose(B.parameters(c), v - 1)
    shared = B.Rx(0.3)
    c2 = B.chain(2, B.put(2, 1, shared), B.put(2, 2, shared))
    assert B.nparameters(c2) == 1
    with pytest.raises(errors.ValidationError):
        B.dispatch(c, [1.0])


def test_dispatch_random_matches_oracle_stream(orc):
    c = C.variational_circuit(4, 2)
    B.dispatch(c, "random")
    assert np.array_equal(B.parameters(c), orc.dispatch_random(B.nparameters(c), 42))


def test_heisenberg_terms():
    t = B.pauli_terms(C.heisenberg(4))
    assert len(t) == 9
    assert all(c == 1 for c, _, _ in t)
    assert len(B.pauli_terms(C.heisenberg(3, periodic=True))) == 9
    # Y·Y on (1,2): coefficient 1, x = z = 0b11
    assert (1, 0b11, 0b11) in [(c, x, z) for c, x, z in t]


def test_pauli_product_algebra():
    # X·Y = iZ on one qubit (chain applies Y first, then X: operator X·Y)
    t = B.pauli_terms(B.chain(1, B.put(1, 1, B.Y), B.put(1, 1, B.X)))
    assert t == [(1j, 0, 1)]


@pytest.mark.parametrize("seed", range(6))
def test_lowering_matches_dense_operator(orc, seed):
    rng = np.random.default_rng(seed)
    n = 4
    blocks = []
    for _ in range(12):
        k = rng.integers(0, 6)
        q = [int(v) for v in rng.permutation(np.arange(1, n + 1))]
        if k == 0:
            blocks.append(B.put(n, q[0], B.Rx(rng.uniform(0, 6))))
        elif k == 1:
            blocks.append(B.control(n, q[1], q[0], B.Ry(rng.uniform(0, 6))))
        elif k == 2:
            blocks.append(B.put(n, (q[0], q[1]), B.rot(B.kron(B.X, B.X), rng.uniform(0, 6))))
        elif k == 3:
            blocks.append(B.control(n, (-q[2], q[1]), q[0], B.shift(rng.uniform(0, 6))))
        elif k == 4:
            blocks.append(B.kron(n, (q[0], B.H), (q[1], B.T)))
        else:
            blocks.append(B.repeat(n, B.Sdag, (q[0], q[2])))
    c = B.chain(n, *blocks)
    st = orc.rand_state(n, 1, seed)
    out = orc.apply_program(st, n, lowered(c), B.parameters(c))
    np.testing.assert_allclose(out[0], B.mat(c) @ st[0], atol=1e-13)
    # dagger
    back = orc.apply_program(out, n, lowered(B.dagger(c)), B.parameters(B.dagger(c)))
    np.testing.assert_allclose(back, st, atol=1e-13)


def test_observable_rejects_non_pauli():
    with pytest.raises(errors.UnsupportedError):
        B.pauli_terms(B.put(2, 1, B.H))


def test_time_evolution_blocks_host():
    """time_evolve / cache structure on the host: the evolution time is a
    parameter, circuits split into gate segments and Krylov steps, dagger negates t."""
    from paper_1912_10877_b200 import blocks as Bk
    from paper_1912_10877_b200 import circuits as Cc
    from paper_1912_10877_b200 import errors as Er
    n = 5
    h = Cc.heisenberg(n)
    te = Bk.time_evolve(Bk.cache(h), 0.25)
    circ = Bk.chain(n, Cc.variational_circuit(n, 1), te, Bk.put(n, 2, Bk.Rx(0.3)))
    assert Bk.nparameters(circ) == Bk.nparameters(Cc.variational_circuit(n, 1)) + 2
    assert [k for k, _ in Bk.segments(circ)] == ["prog", "te", "prog"]
    assert Bk.dagger(te).theta == -0.25
    assert len(Bk.pauli_terms(Bk.cache(h))) == len(Bk.pauli_terms(h))
    import pytest as _pt
    assert not Bk.is_pauli_expression(Bk.put(n, 1, Bk.H))
    Bk.time_evolve(Bk.put(n, 1, Bk.H), 0.1)  # non-Pauli: the sparse (Cached) path
    with _pt.raises(Er.UnsupportedError):
        Bk.time_evolve(Bk.put(20, 1, Bk.H), 0.1)  # too large for a materialised matrix
    with _pt.raises(Er.UnsupportedError):
        Bk.segments(Bk.put(n, (1, 2), Bk.time_evolve(Cc.heisenberg(2), 0.1)))


def test_subroutine_and_qft_host():
    """Subroutine = put on its locations; qft(n) = bit reversal then the inverse DFT
    scaled by sqrt(2^n) (SPEC App F oracle); gatecount(qft(3)) = {H: 3, Control{shift}: 3}."""
    import numpy as np
    import paper_1912_10877_b200 as qb
    s = qb.subroutine(5, qb.dagger(qb.qft(4)), (1, 2, 3, 4))
    assert np.abs(qb.mat(s) - qb.mat(qb.put(5, (1, 2, 3, 4), qb.dagger(qb.qft(4))))).max() == 0.0
    assert qb.gatecount(qb.qft(3)) == {"H": 3, "Control{shift}": 3}
    n = 5
    N = 1 << n
    x = np.random.default_rng(0).normal(size=N) + 1j * np.random.default_rng(1).normal(size=N)
    rev = np.array([int(format(i, f"0{n}b")[::-1], 2) for i in range(N)])
    assert np.abs(qb.mat(qb.qft(n)) @ x - np.fft.ifft(x[rev]) * np.sqrt(N)).max() < 1e-13
