"""Device engine vs the CPU oracle / reference goldens, through the C-ABI (libqbg.so).
Tolerances (north star): complex128 amplitudes, expectations and gradients within 1e-12
relative (norm-wise for states, ‖Δ‖∞/‖ref‖∞ for vectors); complex64 within 1e-5 of the
complex128 oracle relative to the observable scale; measurement bit-exact."""
import numpy as np
import pytest

import oracle as O
import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C
from paper_1912_10877_b200 import matrix as M

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300)


def relinf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def lowered(block):
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    return em


def gate_of(c):
    if c["kind"] == M.MAT_DIAGONAL:
        return M.Diagonal(c["vals"])
    if c["kind"] == M.MAT_PERMUTATION:
        return M.Permutation(c["perm"], c["vals"])
    d = c["dim"]
    return M.Dense(np.asarray(c["vals"]).reshape(d, d).T)


@pytest.fixture(params=[True, False], ids=["fused", "pergate"])
def fusion(request):
    qb.set_fusion(request.param)
    yield request.param
    qb.set_fusion(True)


def test_instruct_reference_goldens(golden):
    for c in golden("instruct_cases.npy"):
        reg = qb.Register(c["n"], c["B"]).set_state(c["inp"])
        qb.instruct(reg, gate_of(c), c["locs"], c["ctrls"], c["cfg"])
        assert rel(reg.state(), c["out"]) < TOL


def test_instruct_t45_reference_goldens(golden, fusion):
    """4- and 5-qubit gates (dense / diagonal / permutation, with controls and batches) through the
    per-gate kernels and the fused engine's fallback, vs the reference's own outputs."""
    for c in golden("instruct_cases_t45.npy"):
        reg = qb.Register(c["n"], c["B"]).set_state(c["inp"])
        qb.instruct(reg, gate_of(c), c["locs"], c["ctrls"], c["cfg"])
        assert rel(reg.state(), c["out"]) < TOL


@pytest.mark.parametrize("tag,params", [("X", ()), ("Y", ()), ("Z", ()), ("H", ()), ("S", ()), ("Sdag", ()),
                                        ("T", ()), ("Tdag", ()), ("I2", ()), ("P0", ()), ("P1", ()), ("Pu", ()),
                                        ("Pd", ()), ("Rx", (0.5,)), ("Ry", (1.1,)), ("Rz", (2.3,)),
                                        ("shift", (0.7,)), ("phase", (0.3,)), ("SWAP", ()), ("CNOT", ()),
                                        ("CZ", ()), ("Toffoli", ())])
def test_instruct_tags_vs_oracle(orc, tag, params):
    n = 7
    t = {"SWAP": 2, "CNOT": 2, "CZ": 2, "Toffoli": 3}.get(tag, 1)
    locs = [3, 6, 1][:t]
    gm = M.CONST_GATES[tag]() if not params else {"Rx": M.rx, "Ry": M.ry, "Rz": M.rz, "shift": M.shift,
                                                  "phase": M.global_phase}[tag](*params)
    st = orc.rand_state(n, 3, 5)
    for ctrls, cfg in [((), ()), ((5,), (1,)), ((5, 7), (0, 1))]:
        want = orc.instruct(st, n, gm, locs, ctrls, cfg)
        reg = qb.Register(n, 3).set_state(st)
        qb.instruct(reg, tag, locs, ctrls, cfg, params)
        assert rel(reg.state(), want) < TOL


def test_instruct_errors():
    reg = qb.zero_state(3)
    with pytest.raises(qb.errors.RangeError):
        qb.instruct(reg, "X", [4])
    with pytest.raises(qb.errors.ValidationError):
        qb.instruct(reg, "SWAP", [1, 1])
    with pytest.raises(qb.errors.ValidationError):
        qb.instruct(reg, "X", [1], [1], [1])
    with pytest.raises(qb.errors.ShapeError):
        qb.instruct(reg, M.swap(), [1])
    with pytest.raises(qb.errors.DispatchError):
        qb.instruct(reg, "Nope", [1])
    with pytest.raises(qb.errors.DispatchError):
        qb.instruct(reg, "Rx", [1])
    with pytest.raises(qb.errors.ResourceError):
        qb.zero_state(qb.qubit_cap() + 1)


@pytest.mark.parametrize("n,depth,nb", [(4, 3, 1), (9, 2, 3), (13, 2, 1), (16, 2, 2)])
def test_program_forward_vs_oracle(orc, fusion, n, depth, nb):
    circ = C.variational_circuit(n, depth)
    th = np.random.default_rng(n).uniform(0, 2 * np.pi, B.nparameters(circ))
    B.dispatch(circ, th)
    st = orc.rand_state(n, nb, 3)
    want = orc.apply_program(st, n, lowered(circ), th)
    reg = qb.Register(n, nb).set_state(st)
    qb.apply(reg, circ)
    assert rel(reg.state(), want) < TOL
    qb.apply(reg, B.dagger(circ))
    assert rel(reg.state(), st) < 1e-11


def test_expect_grad_goldens(golden, fusion):
    g = golden("ad.npz")
    circ = C.variational_circuit(4, 3)
    B.dispatch(circ, g["theta"])
    reg = qb.Register(4, 2).set_state(g["state_in"])
    res = qb.expect_grad(C.heisenberg(4), (reg, circ), want_state_grad=True)
    assert relinf(res.energies, g["energies"]) < TOL
    assert relinf(res.param_grads, g["grads"]) < TOL
    assert rel(res.state_grad.state(), g["state_grad"]) < TOL
    assert rel(reg.state(), g["state_in"]) == 0  # not in place: input untouched


def test_app_g_paper_values(fusion):
    circ = B.chain(B.put(3, 2, B.Rx(0.5)), B.control(3, 2, 1, B.Ry(0.7)),
                   B.put(3, (1, 2), B.rot(B.kron(B.X, B.X), 0.8)))
    res = qb.expect_grad(C.heisenberg(3, periodic=True), (qb.zero_state(3), circ))
    assert abs(res.energies[0] - 1.9542144196547988) < 1e-13
    np.testing.assert_allclose(res.param_grads, [-1.2280830050051128, -0.31110858256435187, -1.5656386306937393],
                               atol=1e-13, rtol=0)


@pytest.mark.parametrize("n,depth,nb", [(6, 2, 1), (11, 2, 4), (14, 1, 1)])
def test_expect_grad_vs_oracle(orc, fusion, n, depth, nb):
    circ = C.variational_circuit(n, depth)
    th = np.random.default_rng(7 * n).uniform(0, 2 * np.pi, B.nparameters(circ))
    B.dispatch(circ, th)
    h = C.heisenberg(n)
    st = orc.rand_state(n, nb, 11)
    e, g, _, sg = orc.expect_grad(st, n, lowered(circ), th, B.pauli_terms(h))
    reg = qb.Register(n, nb).set_state(st)
    res = qb.expect_grad(h, (reg, circ), want_state_grad=True)
    assert relinf(res.energies, e) < TOL
    assert relinf(res.param_grads, g) < TOL
    assert rel(res.state_grad.state(), sg) < TOL
    assert relinf(qb.expect(h, (reg, circ)), e) < TOL


def test_batched_grad_is_sum_of_singles(orc):
    """batched gradients = Σ per-batch gradients (1e-9; we hold 1e-12)."""
    n = 8
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, "random")
    h = C.heisenberg(n)
    st = orc.rand_state(n, 4, 2)
    full = qb.expect_grad(h, (qb.Register(n, 4).set_state(st), circ))
    parts = [qb.expect_grad(h, (qb.Register(n, 1).set_state(st[b:b + 1]), circ)) for b in range(4)]
    assert relinf(full.param_grads, sum(p.param_grads for p in parts)) < TOL
    assert relinf(full.energies, np.concatenate([p.energies for p in parts])) < TOL


def test_uncompute_fidelity_and_constant_memory():
    """in-place expect' restores the input within 1e-10; full-state allocations
    do not grow with depth."""
    n = 10
    h = C.heisenberg(n)
    counts = []
    for depth in (2, 20, 60):
        circ = C.variational_circuit(n, depth)
        B.dispatch(circ, "random")
        reg = qb.rand_state(n, 1, 3)
        before = reg.state()
        a0 = qb.state_alloc_counter()
        qb.expect_grad(h, (reg, circ), inplace=True)
        counts.append(qb.state_alloc_counter() - a0)
        assert rel(reg.state(), before) < 1e-10
    assert counts[1] == counts[2]


def test_measure_bit_exact(golden):
    g = golden("measure.npz")
    reg = qb.Register(6, 2).set_state(g["state"])
    assert np.array_equal(qb.measure(reg, 50, qb.Rng(11)), g["samples"])
    assert np.array_equal(qb.probabilities(reg, 1), g["probs1"])
    hits = qb.measure_collapse(reg, qb.Rng(12))
    assert np.array_equal(hits, g["hits"])
    assert rel(reg.state(), g["collapsed"]) < 1e-15


def test_listing13():
    reg = qb.zero_state(4)
    qb.instruct(reg, "X", [2])
    s = qb.measure(reg, 3)
    assert [qb.to_text(v, 4) for v in s[0]] == ["0010 (2)"] * 3


def test_focus_relax_goldens(golden):
    g = golden("focus.npz")
    locs = [int(v) for v in g["locs"]]
    reg = qb.Register(6, 2).set_state(g["state"])
    reg.focus(locs)
    assert reg.nactive == 4
    assert np.array_equal(reg.state(), g["focused"])
    reg.relax(locs, to_nactive=6)
    assert np.array_equal(reg.state(), g["state"])


def test_focus_then_apply_matches_reference_semantics(orc):
    """focus(3,6,1,2) + H on active qubit 1 + relax == H on qubit 3."""
    st = orc.rand_state(6, 1, 4)
    reg = qb.Register(6).set_state(st)
    reg.focus([3, 6, 1, 2])
    qb.instruct(reg, "H", [1])
    reg.relax([3, 6, 1, 2], to_nactive=6)
    assert rel(reg.state(), orc.instruct(st, 6, M.h(), [3])) < TOL


def test_qbreg1_interchange(tmp_path):
    """Device register <-> QBREG1 file written by the compiled reference (register.hpp:181-205)."""
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, "state_qbreg1.bin")
    amps = np.load(os.path.join(GOLDEN, "state_qbreg1_amps.npy"))
    reg = qb.Register.load(path)
    assert (reg.nqubits, reg.nactive, reg.nbatch) == (4, 3, 2)
    assert np.array_equal(reg.state(), amps)
    reg.save(tmp_path / "o.bin")
    assert open(tmp_path / "o.bin", "rb").read() == open(path, "rb").read()
    with pytest.raises(qb.errors.SerializationError):
        qb.Register.load(os.path.join(GOLDEN, "rng.npz"))


@pytest.mark.parametrize("n", [5, 12])
def test_gradient_triangle(n):
    """reverse mode = parameter shift = central FD (1e-6) — fused path at n = 12."""
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, "random")
    h = C.heisenberg(n)
    reg = qb.zero_state(n)
    rev = qb.expect_grad(h, (reg, circ)).param_grads
    shift = qb.faithful_grad(h, (reg, circ))
    np.testing.assert_allclose(rev, shift, atol=1e-10, rtol=0)
    th = B.parameters(circ)
    for k in range(0, th.size, max(1, th.size // 6)):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-4
        tm[k] -= 1e-4
        B.dispatch(circ, tp)
        ep = qb.expect(h, (reg, circ))[0]
        B.dispatch(circ, tm)
        em = qb.expect(h, (reg, circ))[0]
        assert abs((ep - em) / 2e-4 - rev[k]) < 1e-6
    B.dispatch(circ, th)


def test_register_algebra(orc):
    a = orc.rand_state(9, 3, 1)
    b = orc.rand_state(9, 3, 2)
    ra, rb = qb.Register(9, 3).set_state(a), qb.Register(9, 3).set_state(b)
    np.testing.assert_allclose(ra.inner(rb), orc.inner(a, b), atol=1e-14)
    np.testing.assert_allclose(ra.norm(), np.linalg.norm(a, axis=1), atol=1e-14)
    ra.add_scaled(rb, 0.5 - 0.25j)
    assert rel(ra.state(), a + (0.5 - 0.25j) * b) < 1e-15
    ra.scale(2j)
    assert rel(ra.state(), 2j * (a + (0.5 - 0.25j) * b)) < 1e-15


def test_rand_state_bit_exact(golden):
    g = golden("rng.npz")
    assert np.array_equal(qb.rand_state(5, 3, 42).state(), g["rand_state_5_3_42"])


def test_c64_within_tolerance(orc):
    n = 12
    circ = C.variational_circuit(n, 3)
    B.dispatch(circ, "random")
    h = C.heisenberg(n)
    st = orc.rand_state(n, 1, 8)
    e, g, _, _ = orc.expect_grad(st, n, lowered(circ), B.parameters(circ), B.pauli_terms(h))
    reg = qb.Register(n, 1, dtype="c64").set_state(st)
    res = qb.expect_grad(h, (reg, circ))
    scale = sum(abs(c) for c, _, _ in B.pauli_terms(h))
    assert np.abs(res.energies - e).max() / scale < 1e-5
    assert np.abs(res.param_grads - g).max() / scale < 1e-5


def test_20q_circuit_vs_oracle(orc, fusion):
    n = 20
    circ = C.variational_circuit(n, 1)
    B.dispatch(circ, "random")
    st = orc.rand_state(n, 1, 1)
    want = orc.apply_program(st, n, lowered(circ), B.parameters(circ))
    reg = qb.Register(n).set_state(st)
    qb.apply(reg, circ)
    assert rel(reg.state(), want) < TOL


def test_25q_properties(fusion):
    """At the metric size the oracle is too slow per test: size-independent properties."""
    n = 25
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, "random")
    reg = qb.zero_state(n)
    qb.apply(reg, circ)
    assert abs(reg.norm(0) - 1) < 1e-12
    qb.apply(reg, B.dagger(circ))
    p = qb.probabilities(reg, 0)
    assert abs(p[0] - 1) < 1e-10


def test_one_call_forms(orc):
    """SURVEY §8(b) one-call forms: qbg_run_program / qbg_expect_pauli_sum / qbg_axpy / qbg_collapse
    equal the handle API."""
    import ctypes
    from paper_1912_10877_b200._capi import QbgOp, QbgPauliTerm, check, lib
    n = 12
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, "random")
    th = np.ascontiguousarray(B.parameters(circ))
    em = lowered(circ)
    st = orc.rand_state(n, 2, 8)
    want = qb.Register(n, 2).set_state(st)
    qb.apply(want, circ)
    got = qb.Register(n, 2).set_state(st)
    ops = (QbgOp * len(em.ops))(*em.ops)
    vals = np.ascontiguousarray(np.array(em.vals or [0j], dtype=np.complex128))
    perms = np.ascontiguousarray(np.array(em.perms or [0], dtype=np.int64))
    check(lib().qbg_run_program(got._h, ops, len(em.ops), vals.ctypes.data, len(em.vals), perms.ctypes.data,
                                len(em.perms), th.ctypes.data, th.size))
    assert rel(got.state(), want.state()) < 1e-14
    h = C.heisenberg(n)
    terms = B.pauli_terms(h)
    arr = (QbgPauliTerm * len(terms))(*[QbgPauliTerm(complex(c).real, complex(c).imag, x, z) for c, x, z in terms])
    e = np.empty(2)
    check(lib().qbg_expect_pauli_sum(got._h, arr, len(terms), e.ctypes.data))
    assert relinf(e, qb.expect(h, got)) < 1e-14
    a = got.copy()
    check(lib().qbg_axpy(a._h, got._h, 0.5, -0.25))
    assert rel(a.state(), got.state() * (1.5 - 0.25j)) < 1e-14
    out1 = np.empty(2, dtype=np.uint64)
    out2 = np.empty(2, dtype=np.uint64)
    r1, r2 = got.copy(), got.copy()
    g1, g2 = qb.Rng(5), qb.Rng(5)  # keep the handles alive across the calls
    check(lib().qbg_collapse(r1._h, g1._h, out1.ctypes.data))
    check(lib().qbg_measure_collapse(r2._h, g2._h, out2.ctypes.data))
    assert np.array_equal(out1, out2) and rel(r1.state(), r2.state()) == 0


def test_subroutine_listing16_on_device():
    """Listing 16: inverse QFT on a local scope (Subroutine) equals the explicit focus -> apply ->
    relax of Listing 15, and the put-lowered program; an Add child takes the focus/relax path."""
    st = O.restatement().rand_state(6, 2, 17)
    a = qb.Register(6, 2).set_state(st)
    qb.apply(a, qb.subroutine(6, qb.dagger(qb.qft(4)), (2, 5, 1, 3)))
    b = qb.Register(6, 2).set_state(st)
    b.focus(2, 5, 1, 3)
    qb.apply(b, qb.dagger(qb.qft(4)))
    b.relax(2, 5, 1, 3, to_nactive=6)
    assert rel(a.state(), b.state()) < 1e-14
    want = (qb.mat(qb.put(6, (2, 5, 1, 3), qb.dagger(qb.qft(4)))) @ st.T).T
    assert rel(a.state(), want) < TOL
    obs = qb.subroutine(6, qb.heisenberg(3), (4, 6, 2))
    c = qb.Register(6, 2).set_state(st)
    qb.apply(c, obs)
    assert rel(c.state(), (qb.mat(obs) @ st.T).T) < TOL
