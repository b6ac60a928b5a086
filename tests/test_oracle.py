"""The CPU oracle restatement, pinned against the compiled reference's golden fixtures
(tests/golden/make_golden.py) and the paper's / SPEC's known answers.  CPU only."""
import numpy as np
import pytest

import oracle as O
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C
from paper_1912_10877_b200 import matrix as M


def gate_of(c):
    if c["kind"] == M.MAT_DIAGONAL:
        return M.Diagonal(c["vals"])
    if c["kind"] == M.MAT_PERMUTATION:
        return M.Permutation(c["perm"], c["vals"])
    d = c["dim"]
    return M.Dense(np.asarray(c["vals"]).reshape(d, d).T)


def lowered(block):
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    return em


def test_instruct_matches_reference_goldens(orc, golden):
    cases = golden("instruct_cases.npy")
    assert len(cases) >= 200
    for c in cases:
        out = orc.instruct(c["inp"], c["n"], gate_of(c), c["locs"], c["ctrls"], c["cfg"])
        # same formulas, same libstdc++, -ffp-contract=off: bit-exact
        assert np.array_equal(out, c["out"]), (c["n"], c["locs"], c["ctrls"])


def test_instruct_t45_goldens_bit_exact(orc, golden):
    """4- and 5-qubit gates (the widest dense blocks, register.hpp:371-384), reference-generated."""
    cases = golden("instruct_cases_t45.npy")
    assert len(cases) >= 60 and {len(c["locs"]) for c in cases} == {4, 5}
    for c in cases:
        out = orc.instruct(c["inp"], c["n"], gate_of(c), c["locs"], c["ctrls"], c["cfg"])
        assert np.array_equal(out, c["out"]), (c["n"], c["locs"], c["ctrls"])


def test_rng_and_rand_state_bit_exact(orc, golden):
    g = golden("rng.npz")
    r = orc.rng(42)
    assert np.array_equal([r.uniform() for _ in range(64)], g["uniform"])
    assert np.array_equal(np.array([r.bits() for _ in range(16)], dtype=np.uint64), g["bits"])
    assert np.array_equal([r.gauss() for _ in range(32)], g["gauss"])
    assert np.array_equal(orc.dispatch_random(75, 42), g["dispatch_random"])
    assert np.array_equal(orc.rand_state(5, 3, 42), g["rand_state_5_3_42"])


def test_expect_grad_goldens(orc, golden):
    g = golden("ad.npz")
    circ = C.variational_circuit(4, 3)
    B.dispatch(circ, g["theta"])
    em = lowered(circ)
    e, gr, psi, sg = orc.expect_grad(g["state_in"], 4, em, g["theta"], B.pauli_terms(C.heisenberg(4)))
    np.testing.assert_allclose(e, g["energies"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(gr, g["grads"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(psi, g["psi_back"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(sg, g["state_grad"], rtol=0, atol=1e-13)
    fwd = orc.apply_program(g["state_in"], 4, em, g["theta"])
    assert np.array_equal(fwd, g["forward"])


def test_app_g_paper_values(orc):
    """PAPER.md:1424-1474 (periodic heisenberg(3), App G): E and the three gradients."""
    circ = B.chain(B.put(3, 2, B.Rx(0.5)), B.control(3, 2, 1, B.Ry(0.7)),
                   B.put(3, (1, 2), B.rot(B.kron(B.X, B.X), 0.8)))
    e, g, _, _ = orc.expect_grad(O.Oracle.zero_state(3), 3, lowered(circ), B.parameters(circ),
                                 B.pauli_terms(C.heisenberg(3, periodic=True)))
    assert abs(e[0] - 1.9542144196547988) < 1e-14
    np.testing.assert_allclose(g, [-1.2280830050051128, -0.31110858256435187, -1.5656386306937393],
                               rtol=0, atol=1e-14)


def test_spec_examples(orc):
    # <Z> after Rx(0.4) on |0> = cos 0.4 ; dθ = -sin 0.4
    circ = B.chain(B.put(1, 1, B.Rx(0.4)))
    z = B.put(1, 1, B.Z)
    e, g, _, _ = orc.expect_grad(O.Oracle.zero_state(1), 1, lowered(circ), [0.4], B.pauli_terms(z))
    assert abs(e[0] - np.cos(0.4)) < 1e-15 and abs(g[0] + np.sin(0.4)) < 1e-15
    # expect(heisenberg(2), |00>) = 1
    _, e2 = orc.obs_apply(O.Oracle.zero_state(2), B.pauli_terms(C.heisenberg(2)))
    assert e2[0] == 1.0


def test_listing13_measure(orc):
    """Listing 13 / SPEC.md:235: instruct X on qubit 2 of zero_state(4), three shots -> 0010."""
    st = orc.instruct(O.Oracle.zero_state(4), 4, M.x(), [2])
    s = orc.measure(st, 4, 4, 3, orc.rng(42))
    assert s.tolist() == [[2, 2, 2]]


def test_measure_goldens(orc, golden):
    g = golden("measure.npz")
    assert np.array_equal(orc.measure(g["state"], 6, 6, 50, orc.rng(11)), g["samples"])
    hits, col = orc.measure_collapse(g["state"], 6, 6, orc.rng(12))
    assert np.array_equal(hits, g["hits"]) and np.array_equal(col, g["collapsed"])
    assert np.array_equal(orc.probabilities(g["state"], 6, 6, 1), g["probs1"])


def test_focus_relax_goldens(orc, golden):
    g = golden("focus.npz")
    locs = [int(v) for v in g["locs"]]
    f = orc.focus(g["state"], 6, locs)
    assert np.array_equal(f, g["focused"])
    assert np.array_equal(orc.relax(f, 6, locs), g["state"])


def test_qbreg1_interchange(orc, golden, tmp_path):
    """register.hpp:181-205: the file the reference wrote loads bit-exactly; ours is byte-identical."""
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, "state_qbreg1.bin")
    amps = np.load(os.path.join(GOLDEN, "state_qbreg1_amps.npy"))
    st, n, na = orc.load(path)
    assert (n, na) == (4, 3) and np.array_equal(st, amps)
    out = tmp_path / "o.bin"
    orc.save(amps, 4, 3, out)
    assert open(out, "rb").read() == open(path, "rb").read()


def test_validation_order(orc):
    st = O.Oracle.zero_state(3)
    with pytest.raises(O.OracleError) as e:
        orc.instruct(st, 3, M.x(), [4])
    assert e.value.code == 3  # RangeError
    with pytest.raises(O.OracleError) as e:
        orc.instruct(st, 3, M.swap(), [1, 1])
    assert e.value.code == 1  # ValidationError (duplicate target)
    with pytest.raises(O.OracleError) as e:
        orc.instruct(st, 3, M.x(), [1], [1], [1])
    assert e.value.code == 1  # control overlaps
    with pytest.raises(O.OracleError) as e:
        orc.instruct(st, 3, M.swap(), [1])
    assert e.value.code == 2  # ShapeError


def test_restatement_matches_reference_fresh_cases(orc, ref):
    rng = np.random.default_rng(99)
    for _ in range(50):
        n = int(rng.integers(2, 8))
        circ = C.variational_circuit(n, int(rng.integers(1, 3)))
        th = rng.uniform(0, 2 * np.pi, B.nparameters(circ))
        B.dispatch(circ, th)
        em = lowered(circ)
        st = orc.rand_state(n, 2, int(rng.integers(0, 1000)))
        a = orc.apply_program(st, n, em, th)
        b = ref.apply_program(st, n, em, th)
        assert np.array_equal(a, b)
        terms = B.pauli_terms(C.heisenberg(n))
        ea, ga, _, _ = orc.expect_grad(st, n, em, th, terms)
        eb, gb, _, _ = ref.expect_grad(st, n, em, th, terms)
        np.testing.assert_allclose(ea, eb, atol=1e-14, rtol=0)
        np.testing.assert_allclose(ga, gb, atol=1e-13, rtol=0)


@pytest.mark.parametrize("seed", range(5))
def test_gradient_triangle_oracle(orc, seed):
    """reverse-mode = central finite differences (eps 1e-4) within 1e-6."""
    circ = C.variational_circuit(4, 3)
    th = np.random.default_rng(seed).uniform(0, 2 * np.pi, B.nparameters(circ))
    em = lowered(circ)
    terms = B.pauli_terms(C.heisenberg(4))
    st = O.Oracle.zero_state(4)
    _, g, _, _ = orc.expect_grad(st, 4, em, th, terms)
    fd = np.empty_like(th)
    for k in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-4
        tm[k] -= 1e-4
        ep = orc.obs_apply(orc.apply_program(st, 4, em, tp), terms)[1][0]
        emn = orc.obs_apply(orc.apply_program(st, 4, em, tm), terms)[1][0]
        fd[k] = (ep - emn) / 2e-4
    np.testing.assert_allclose(g, fd, atol=1e-6, rtol=0)


def test_mmd_oracle_zero_and_fd(orc):
    """The dense MMD restatement (oracle.mmd_dense): L = 0 at p = q, L >= 0,
    and its reverse-mode gradient (oracle backward) equals central finite differences."""
    from paper_1912_10877_b200.mmd import brbf_kernel
    n = 4
    circ = C.variational_circuit(n, 2)
    th = np.random.default_rng(3).uniform(0, 2 * np.pi, B.nparameters(circ))
    B.dispatch(circ, th)
    st = orc.zero_state(n)
    q = np.random.default_rng(5).uniform(0, 1, 1 << n)
    q /= q.sum()
    psi = orc.apply_program(st, n, lowered(circ), th)
    p = np.abs(psi[0]) ** 2
    assert abs(O.mmd_dense(psi, p / p.sum(), [2.0])[0][0]) < 1e-15
    L, g = O.mmd_grad_dense(orc, st, n, lowered(circ), th, q, [2.0, 0.7])
    assert L[0] >= 0
    for k in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-5
        tm[k] -= 1e-5
        lp = O.mmd_dense(orc.apply_program(st, n, lowered(circ), tp), q, [2.0, 0.7])[0][0]
        lm = O.mmd_dense(orc.apply_program(st, n, lowered(circ), tm), q, [2.0, 0.7])[0][0]
        assert abs((lp - lm) / 2e-5 - g[k]) < 1e-7
    kf = brbf_kernel(2.0, 0.7)
    assert np.isclose(kf(3, 5), np.exp(-4 / 8) + np.exp(-4 / (2 * 0.49)))
    with pytest.raises(Exception):
        brbf_kernel(-1.0)


def test_pauli_dense_matches_oracle_obs_apply(orc):
    """The dense Hamiltonian used as the time-evolution oracle applies like orc_obs_apply."""
    from paper_1912_10877_b200 import blocks as Bk
    n = 5
    st = orc.rand_state(n, 2, 3)
    for blk in (C.heisenberg(n), Bk.kron(n, ((1,), Bk.Y), ((4,), Bk.Y), ((2,), Bk.Z))):
        t = Bk.pauli_terms(blk)
        H = O.pauli_dense(t, n)
        phi, _ = orc.obs_apply(st, t)
        assert np.abs(phi - (H @ st.T).T).max() < 1e-14
        assert np.abs(H - H.conj().T).max() == 0
    U = O.expm_apply(np.eye(1 << 3), Bk.pauli_terms(C.heisenberg(3)), 3, 0.4)
    assert np.abs(U @ U.conj().T - np.eye(8)).max() < 1e-13
