"""The checkpointed expect': the forward passes keep the state after every reverse
segment, the reverse passes read ψ from those checkpoints and take all of a pass's gradient
statistics first.  Checked here against the uncompute design (the same engine with
qbg_set_checkpointing(0)), which test_gpu_parity / test_gpu_random_circuits / test_gpu_bench_parity
pin to the CPU oracle and the reference's goldens — those suites run the checkpointed path by
default (every register of >= 11 qubits whose checkpoints fit).  Also: the register is never
modified, the checkpoint plans are the ones that ran, and a register too large for its checkpoints
falls back to the uncompute design."""
import numpy as np
import pytest

import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B

from test_gpu_random_circuits import random_circuit

pytestmark = pytest.mark.gpu


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300)


def both(obs, make_reg, circ, want_state_grad=False, inplace=False):
    out = []
    for on in (True, False):
        qb.set_checkpointing(on)
        try:
            r = qb.expect_grad(obs, (make_reg(), circ), want_state_grad=want_state_grad, inplace=inplace)
            qb.synchronize()
        finally:
            qb.set_checkpointing(True)
        out.append(r)
    return out


@pytest.mark.parametrize("n,d,nb", [(12, 2, 1), (14, 4, 1), (13, 3, 4), (16, 6, 2)])
def test_variational_matches_uncompute(n, d, nb):
    c = qb.variational_circuit(n, d)
    qb.dispatch(c, np.random.default_rng(n * 7 + d).uniform(0, 2 * np.pi, qb.nparameters(c)))
    h = qb.heisenberg(n)
    ck, un = both(h, lambda: qb.rand_state(n, nbatch=nb, seed=5), c, want_state_grad=True)
    assert relerr(ck.energies, un.energies) < 1e-12
    assert relerr(ck.param_grads, un.param_grads) < 1e-12
    assert relerr(ck.state_grad.state(), un.state_grad.state()) < 1e-12


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_circuits_match_uncompute(seed):
    """Controlled rotations (scalar-gradient statistics: the stage-layout prologue), diagonal runs,
    2-qubit rotations and dense blocks."""
    n = 13
    c = random_circuit(n, 120, seed)
    ck, un = both(qb.heisenberg(n, periodic=True), lambda: qb.rand_state(n, seed=seed), c)
    assert relerr(ck.energies, un.energies) < 1e-12
    assert relerr(ck.param_grads, un.param_grads) < 1e-11


def test_c64_matches_uncompute():
    n = 14
    c = qb.variational_circuit(n, 3)
    qb.dispatch(c, "random")
    ck, un = both(qb.heisenberg(n), lambda: qb.zero_state(n, dtype="c64"), c)
    assert relerr(ck.param_grads, un.param_grads) < 1e-5


@pytest.mark.parametrize("inplace", [False, True])
def test_register_unmodified(inplace):
    n = 13
    c = qb.variational_circuit(n, 3)
    qb.dispatch(c, "random")
    reg = qb.rand_state(n, nbatch=2, seed=9)
    before = reg.state().copy()
    qb.expect_grad(qb.heisenberg(n), (reg, c), inplace=inplace)
    qb.synchronize()
    assert np.array_equal(reg.state(), before)  # bit-exact: the checkpointed path never writes it


def test_checkpoint_plans_ran():
    n = 15
    c = qb.variational_circuit(n, 3)
    qb.dispatch(c, "random")
    qb.expect_grad(qb.heisenberg(n), (qb.zero_state(n), c))
    qb.synchronize()
    info = B.compile_block(c).plan_info()
    assert "plan dir=5" in info and "plan dir=4" in info, info
    # the mirror forward plan has one segment per reverse step: equal step counts
    steps = {ln.split()[1]: int(ln.split("steps=")[1].split()[0]) for ln in info.splitlines() if ln.startswith("plan dir=")}
    assert steps["dir=4"] >= steps["dir=5"] > 0


def test_repeated_steps_and_new_theta():
    """An optimiser loop: new θ every step (values-only refresh of both checkpoint plans)."""
    n = 12
    c = qb.variational_circuit(n, 3)
    h = qb.heisenberg(n)
    rng = np.random.default_rng(4)
    for _ in range(3):
        qb.dispatch(c, rng.uniform(0, 2 * np.pi, qb.nparameters(c)))
        ck, un = both(h, lambda: qb.zero_state(n), c)
        assert relerr(ck.param_grads, un.param_grads) < 1e-12


def test_mmd_loss_matches_uncompute():
    n = 12
    c = qb.variational_circuit(n, 2)
    qb.dispatch(c, "random")
    target = np.random.default_rng(3).random(1 << n)
    target /= target.sum()
    mmd = qb.MMD(qb.brbf_kernel(0.25, 4.0), target)
    ck, un = both(mmd, lambda: qb.zero_state(n), c)
    assert relerr(ck.energies, un.energies) < 1e-12
    assert relerr(ck.param_grads, un.param_grads) < 1e-11


def test_over_limit_falls_back_to_uncompute():
    """Checkpoints that do not fit (here: a 1-byte limit) -> the uncompute design runs, same result."""
    n = 13
    c = qb.variational_circuit(n, 3)
    qb.dispatch(c, "random")
    h = qb.heisenberg(n)
    ref = qb.expect_grad(h, (qb.zero_state(n), c))
    qb.set_checkpoint_limit(1)
    try:
        reg = qb.zero_state(n)
        r = qb.expect_grad(h, (reg, c), inplace=True)
        qb.synchronize()
    finally:
        qb.set_checkpoint_limit(-1)
    assert relerr(r.param_grads, ref.param_grads) < 1e-12
    assert "plan dir=2" in B.compile_block(c).plan_info()
    # the uncompute design leaves the in-place register uncomputed back to |0> up to rounding
    z = np.zeros(1 << n, complex)
    z[0] = 1
    assert relerr(reg.state().ravel(), z) < 1e-12
