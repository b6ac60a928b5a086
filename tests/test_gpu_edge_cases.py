"""Edge cases of the device engine vs the CPU oracle, through the C-ABI: the smallest registers
(1-2 qubits, below the 3 coalescing qubits of a tile), an empty circuit, registers at and around
the tile sizes (2^10 / 2^11 / 2^12 elements) where the planner switches between the per-gate
and the tiled passes, wide batches of tiny states, and run-to-run determinism of the gradient
reductions (fixed reduction order).  Tolerances as in test_gpu_parity.py."""
import numpy as np
import pytest

import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C

pytestmark = pytest.mark.gpu

TOL = 1e-12


def relinf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.size == 0 and b.size == 0:
        return 0.0
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300)


def lowered(block):
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    return em


@pytest.fixture(params=[True, False], ids=["fused", "pergate"])
def fusion(request):
    qb.set_fusion(request.param)
    yield request.param
    qb.set_fusion(True)


def check_expect_grad(orc, n, circ, obs, nb, seed=5):
    st = orc.rand_state(n, nb, seed)
    e, g, _, sg = orc.expect_grad(st, n, lowered(circ), B.parameters(circ), B.pauli_terms(obs))
    reg = qb.Register(n, nb).set_state(st)
    res = qb.expect_grad(obs, (reg, circ), want_state_grad=True)
    assert relinf(res.energies, e) < TOL
    assert relinf(res.param_grads, g) < TOL
    assert rel(res.state_grad.state(), sg) < TOL
    return res


@pytest.mark.parametrize("nb", [1, 3])
def test_one_qubit_register(orc, fusion, nb):
    circ = B.chain(B.put(1, 1, B.Rx(0.3)), B.put(1, 1, B.Rz(0.7)), B.put(1, 1, B.Ry(-1.1)),
                   B.put(1, 1, B.shift(0.4)), B.put(1, 1, B.H))
    check_expect_grad(orc, 1, circ, B.put(1, 1, B.Z), nb)
    check_expect_grad(orc, 1, circ, B.Add([B.put(1, 1, B.X), B.Scale(0.5, B.put(1, 1, B.Y))]), nb)


@pytest.mark.parametrize("nb", [1, 2])
def test_two_qubit_register(orc, fusion, nb):
    circ = C.variational_circuit(2, 3)
    B.dispatch(circ, np.random.default_rng(2).uniform(0, 2 * np.pi, B.nparameters(circ)))
    check_expect_grad(orc, 2, circ, C.heisenberg(2), nb)


def test_empty_circuit(orc, fusion):
    n = 5
    circ = B.chain(n)
    assert B.nparameters(circ) == 0
    reg = qb.Register(n, 2).set_state(orc.rand_state(n, 2, 1))
    before = reg.state()
    qb.apply(reg, circ)
    assert np.array_equal(reg.state(), before)  # identity, bit for bit
    res = check_expect_grad(orc, n, circ, C.heisenberg(n), 2, seed=1)
    assert res.param_grads.shape == (0,)


@pytest.mark.parametrize("n", [10, 11, 12])
def test_tile_boundary_sizes(orc, fusion, n):
    circ = C.variational_circuit(n, 1)
    B.dispatch(circ, np.random.default_rng(n).uniform(0, 2 * np.pi, B.nparameters(circ)))
    check_expect_grad(orc, n, circ, C.heisenberg(n), 1, seed=n)


def test_wide_batch_of_tiny_states(orc, fusion):
    n, nb = 3, 64
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, np.random.default_rng(9).uniform(0, 2 * np.pi, B.nparameters(circ)))
    check_expect_grad(orc, n, circ, C.heisenberg(n, periodic=True), nb, seed=9)


def test_gradients_are_deterministic():
    """Same inputs, same grid: the two-level gradient reductions run in a fixed order, so repeated
    runs agree bit for bit (no atomics on the gradient path)."""
    n = 16
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, np.random.default_rng(4).uniform(0, 2 * np.pi, B.nparameters(circ)))
    h = C.heisenberg(n)
    runs = [qb.expect_grad(h, (qb.zero_state(n), circ)) for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(r.energies, runs[0].energies)
        assert np.array_equal(r.param_grads, runs[0].param_grads)


def _mixed_circuit(n, th):
    """Every parameterised generator kind the engine realises: rotations with diagonal (Z, ZZ),
    permutation (X, XX) and dense (Y) generators, shift, phase, controlled rotations."""
    it = iter(th)
    return B.chain(
        B.put(n, 1, B.Rx(next(it))), B.put(n, 2, B.Ry(next(it))), B.put(n, 3, B.Rz(next(it))),
        B.put(n, (1, 2), B.rot(B.kron(B.X, B.X), next(it))), B.put(n, (2, 3), B.rot(B.kron(B.Z, B.Z), next(it))),
        B.put(n, 4, B.shift(next(it))), B.put(n, 1, B.phase(next(it))),
        B.control(n, 2, 4, B.Rx(next(it))), B.control(n, (1, 3), 5, B.Ry(next(it))),
        B.put(n, 5, B.H),
        B.put(n, 3, B.rot(B.Y, next(it))))


def test_redispatch_matches_fresh_program():
    """dispatch() on a compiled program refreshes only the parameterised ops' matrices in place
    (capi.cu realise_params); the results must equal a freshly compiled program's bit for bit."""
    n = 12
    rng = np.random.default_rng(21)
    th1, th2 = rng.uniform(0, 2 * np.pi, 10), rng.uniform(0, 2 * np.pi, 10)
    h = C.heisenberg(n)
    reused = _mixed_circuit(n, th1)
    qb.expect_grad(h, (qb.zero_state(n), reused))  # realised at th1
    B.dispatch(reused, th2)
    fresh = _mixed_circuit(n, th2)
    for fusion in (True, False):
        qb.set_fusion(fusion)
        try:
            a = qb.expect_grad(h, (qb.zero_state(n), reused), want_state_grad=True)
            b = qb.expect_grad(h, (qb.zero_state(n), fresh), want_state_grad=True)
            r1, r2 = qb.zero_state(n), qb.zero_state(n)
            qb.apply(r1, reused)
            qb.apply(r2, fresh)
        finally:
            qb.set_fusion(True)
        assert np.array_equal(a.energies, b.energies)
        assert np.array_equal(a.param_grads, b.param_grads)
        assert np.array_equal(a.state_grad.state(), b.state_grad.state())
        assert np.array_equal(r1.state(), r2.state())


@pytest.mark.parametrize("dtype,nbatch", [("c128", 1), ("c128", 4), ("c64", 2)])
def test_plan_value_refresh_over_many_thetas(dtype, nbatch):
    """A new θ on a program whose fused plans exist rewrites only the plans' matrix values
    (fused.cu refresh_values: same passes, ops and kernels).  Over successive θ — an optimiser
    loop — the reused program must match a freshly compiled one bit for bit, forward and reverse."""
    n, d = 13, 3
    h = C.heisenberg(n)
    reused = C.variational_circuit(n, d)
    rng = np.random.default_rng(5)
    P = B.nparameters(reused)
    for it in range(4):
        th = rng.uniform(0, 2 * np.pi, P)
        if it == 2:
            th[::7] = 0.0  # rotations at the identity keep their structure
        B.dispatch(reused, th)
        fresh = C.variational_circuit(n, d)
        B.dispatch(fresh, th)
        a = qb.expect_grad(h, (qb.zero_state(n, nbatch=nbatch, dtype=dtype), reused))
        b = qb.expect_grad(h, (qb.zero_state(n, nbatch=nbatch, dtype=dtype), fresh))
        assert np.array_equal(a.energies, b.energies)
        assert np.array_equal(a.param_grads, b.param_grads)
        r1, r2 = qb.zero_state(n, nbatch=nbatch, dtype=dtype), qb.zero_state(n, nbatch=nbatch, dtype=dtype)
        qb.apply(r1, reused)
        qb.apply(r2, fresh)
        assert np.array_equal(r1.state(), r2.state())


@pytest.mark.parametrize("dtype,nbatch", [("c128", 1), ("c128", 2), ("c64", 4)])
def test_out_of_place_expect_grad_reads_input_directly(dtype, nbatch):
    """The out-of-place expect' starts with a forward pass that loads the caller's register and
    stores the work state (no device copy first).  The input must be left untouched, and the
    results must equal the in-place run's bit for bit (the same passes on the same values)."""
    n = 13
    circ = C.variational_circuit(n, 3)
    B.dispatch(circ, np.random.default_rng(8).uniform(0, 2 * np.pi, B.nparameters(circ)))
    h = C.heisenberg(n)
    reg = qb.rand_state(n, nbatch, seed=4, dtype=dtype)
    before = reg.state().copy()
    a = qb.expect_grad(h, (reg, circ))
    assert np.array_equal(reg.state(), before)
    b = qb.expect_grad(h, (reg.copy(), circ), inplace=True)
    assert np.array_equal(a.energies, b.energies)
    assert np.array_equal(a.param_grads, b.param_grads)
