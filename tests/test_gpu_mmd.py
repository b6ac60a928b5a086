"""MMD loss (§3.2, Listing 12) on the device
vs the dense oracle restatement (oracle.mmd_dense / mmd_grad_dense) through the C-ABI.
Tolerance: 1e-12 relative (complex128; the device sums the Toeplitz band in a different order)."""
import numpy as np
import pytest

import oracle as O
import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B
from paper_1912_10877_b200 import circuits as C
from paper_1912_10877_b200 import errors

from test_gpu_parity import lowered, relinf

pytestmark = pytest.mark.gpu

TOL = 1e-12


def target(n, seed=42):
    q = np.random.default_rng(seed).uniform(0, 1, 1 << n)
    return q / q.sum()


@pytest.mark.parametrize("n,nb,sigmas", [(5, 1, [2.0]), (8, 3, [0.5, 2.0, 7.0]), (11, 1, [2.0]), (10, 40, [1.5])])
def test_mmd_loss_and_seed_vs_dense(orc, n, nb, sigmas):
    st = orc.rand_state(n, nb, 3)
    q = target(n)
    L, phi = O.mmd_dense(st, q, sigmas)
    loss = qb.MMD(qb.brbf_kernel(*sigmas), q)
    reg = qb.Register(n, nb).set_state(st)
    assert relinf(qb.mmd_expect(loss, reg), L) < TOL
    vals, adj = qb.mmd_seed(loss, reg)
    assert relinf(vals, L) < TOL
    assert relinf(adj.state(), phi) < TOL


def test_mmd_zero_when_p_equals_target(orc):
    n = 7
    st = orc.rand_state(n, 1, 5)
    q = np.abs(st[0]) ** 2
    q = q / q.sum()
    loss = qb.MMD(qb.brbf_kernel(2.0), q)
    assert abs(qb.mmd_expect(loss, qb.Register(n, 1).set_state(st))[0]) < 1e-15


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("n,depth,nb", [(5, 2, 1), (9, 2, 2), (12, 1, 1)])
def test_mmd_reverse_grad_vs_oracle(orc, fused, n, depth, nb):
    qb.set_fusion(fused)
    try:
        circ = C.variational_circuit(n, depth)
        th = np.random.default_rng(n).uniform(0, 2 * np.pi, B.nparameters(circ))
        B.dispatch(circ, th)
        st = orc.rand_state(n, nb, 9)
        q = target(n, 1)
        L, g = O.mmd_grad_dense(orc, st, n, lowered(circ), th, q, [2.0])
        loss = qb.MMD(qb.brbf_kernel(2.0), q)
        res = qb.expect_grad(loss, (qb.Register(n, nb).set_state(st), circ))
        assert relinf(res.energies, L) < TOL
        assert relinf(res.param_grads, g) < 1e-11
    finally:
        qb.set_fusion(True)


def test_mmd_shift_equals_reverse_and_fd():
    """shift-mode = reverse-mode (1e-6) and FD (1e-6), 3 qubits depth 2."""
    n = 3
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, "random", rng=qb.Rng(42))
    q = target(n, 4)
    loss = qb.MMD(qb.brbf_kernel(2.0), q)
    reg = qb.zero_state(n)
    rev = qb.mmd_grad(loss, (reg, circ), mode="reverse").param_grads
    sh = qb.mmd_grad(loss, (reg, circ), mode="shift").param_grads
    np.testing.assert_allclose(sh, rev, atol=1e-12, rtol=0)
    th = B.parameters(circ)
    for k in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-5
        tm[k] -= 1e-5
        B.dispatch(circ, tp)
        lp = qb.expect(loss, (reg, circ))[0]
        B.dispatch(circ, tm)
        lm = qb.expect(loss, (reg, circ))[0]
        assert abs((lp - lm) / 2e-5 - rev[k]) < 1e-6
    B.dispatch(circ, th)
    assert np.allclose(qb.faithful_grad(loss, (reg, circ)), rev, atol=1e-12)


def test_listing12_shape():
    """Listing 12: g_reg, g_params = expect'(mmd, zero_state(5)=>circuit)."""
    n = 5
    circ = C.variational_circuit(n, 2)
    B.dispatch(circ, "random")
    q = target(n, 7)
    mmd = qb.MMD(qb.brbf_kernel(2.0), q)
    r = qb.expect_grad(mmd, (qb.zero_state(n), circ), want_state_grad=True)
    assert r.param_grads.shape == (B.nparameters(circ),)
    assert r.state_grad.nqubits == n
    assert r.energies[0] >= 0.0


def test_mmd_errors():
    with pytest.raises(errors.ValidationError):
        qb.MMD(qb.brbf_kernel(2.0), np.full(8, 0.2))  # sums to 1.6
    with pytest.raises(errors.ValidationError):
        qb.MMD(qb.brbf_kernel(2.0), np.array([1.5, -0.5]))
    loss = qb.MMD(qb.brbf_kernel(2.0), np.full(8, 0.125))
    with pytest.raises(errors.ShapeError):
        qb.mmd_expect(loss, qb.zero_state(4))
    assert loss.band == 7  # clamped to the basis size
    assert qb.MMD(qb.brbf_kernel(2.0), np.full(256, 1 / 256)).band == 77  # exp(-k^2/8) == 0.0 from k = 78


def test_mmd_20q_band_matches_dense_sample(orc):
    """cfg 3 MMD variant size (2^20 outcomes): spot-check (K d)_x at random rows from the seed."""
    n = 20
    reg = qb.rand_state(n, 1, seed=3)
    q = target(n, 42)
    loss = qb.MMD(qb.brbf_kernel(2.0), q)
    vals, adj = qb.mmd_seed(loss, reg)
    psi = reg.state()[0]
    a = adj.state()[0]
    d = np.abs(psi) ** 2 - q
    rows = np.random.default_rng(0).integers(0, 1 << n, 64)
    for x in list(rows) + [0, (1 << n) - 1]:
        lo, hi = max(0, x - 100), min(1 << n, x + 101)
        ks = np.arange(lo, hi)
        kd = np.sum(np.exp(-((ks - x) ** 2) / 8.0) * d[lo:hi])
        assert abs(a[x] - 2 * kd * psi[x]) <= 1e-12 * max(abs(2 * kd * psi[x]), 1e-30) + 1e-300
