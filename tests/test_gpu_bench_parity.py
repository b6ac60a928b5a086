"""Parity pinned AT THE BENCHMARKED CONFIGURATIONS, against fixtures the compiled reference
wrote (tests/golden/make_golden_bench.py; oracle/_ref = the unmodified /root/reference headers).

  * the metric run of bench.py itself: expect'(heisenberg(25) open, zero_state(25) =>
    variational_circuit(25,10)), θ from Rng(42) — energy, all 775 gradients, 64 amplitudes of ψ_N;
  * variational_circuit(16,10) / (20,10) apply+grad;
  * the cfg-3 shape: 12 qubits x B = 1000 product states, gradient summed over the batch;
  * a cfg-4-sized state: 28 qubits, variational_circuit(28,1) forward + <heisenberg(28)>.

Tolerance (north star): 1e-12, as ‖Δ‖∞ / max(1, ‖ref‖∞) for energies and gradient
vectors (the observable scale bounds |E|), norm-wise relative for amplitudes."""
import numpy as np
import pytest

import paper_1912_10877_b200 as qb

pytestmark = pytest.mark.gpu

TOL = 1e-12


def vec_err(got, want):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    return np.abs(got - want).max() / max(1.0, np.abs(want).max())


def amp_err(got, want):
    return np.linalg.norm(got - want) / np.linalg.norm(want)


def bench_circuit(n, d, theta):
    circ = qb.variational_circuit(n, d)
    qb.dispatch(circ, "random", rng=qb.Rng(42))  # exactly bench.py's stream (rank 0)
    got = qb.parameters(circ)
    assert np.array_equal(got, theta), "dispatch('random') stream differs from the reference's Rng(42)"
    return circ


def test_bench25_metric_run_vs_reference(golden):
    """THE benchmarked step (bench.py default) against the reference's full apply+grad."""
    g = golden("bench25.npz")
    n, d = 25, 10
    circ = bench_circuit(n, d, g["theta"])
    h = qb.heisenberg(n)
    res = qb.expect_grad(h, (qb.zero_state(n), circ))
    e_err, g_err = vec_err(res.energies, g["energy"]), vec_err(res.param_grads, g["grads"])
    print(f"25q d10: |dE| {e_err:.2e}  |dgrad|inf {g_err:.2e}")
    assert res.param_grads.shape == (775,)
    assert e_err <= TOL and g_err <= TOL
    # ψ_N amplitudes (forward only) at 64 fixed indices, and its norm
    reg = qb.zero_state(n)
    qb.apply(reg, circ)
    st = reg.state()[0]
    assert amp_err(st[g["probe_idx"]], g["probes"]) <= TOL
    assert abs(float(np.vdot(st, st).real) - float(g["norm2"])) <= 1e-12


@pytest.mark.parametrize("n", [16, 20])
def test_variational_depth10_vs_reference(golden, n):
    g = golden("bench_small.npz")
    circ = bench_circuit(n, 10, g[f"q{n}_theta"])
    res = qb.expect_grad(qb.heisenberg(n), (qb.zero_state(n), circ))
    assert vec_err(res.energies, g[f"q{n}_energy"]) <= TOL
    assert vec_err(res.param_grads, g[f"q{n}_grads"]) <= TOL


def test_batched_product_states_cfg3_shape(golden):
    """cfg 3's shape: B = 1000 product states (bits from Rng(42)), batch-innermost on the device;
    energies per batch and the gradient summed over the batch."""
    g = golden("bench_small.npz")
    n = 12
    bits = [int(b) for b in g["batch_bits"]]
    r = qb.Rng(42)
    assert bits == [r.bits() & ((1 << n) - 1) for _ in range(1000)]
    circ = bench_circuit(n, 10, g["batch_theta"])
    reg = qb.product_state(bits, nbits=n)
    assert reg.nbatch == 1000
    res = qb.expect_grad(qb.heisenberg(n), (reg, circ))
    assert vec_err(res.energies, g["batch_energies"]) <= TOL
    assert vec_err(res.param_grads, g["batch_grads"]) <= TOL


def test_28q_state_vs_reference(golden):
    """A cfg-4-sized register (4 GiB): the 2^11-tile planner at 28 qubits, forward + energy."""
    g = golden("cfg4_28q.npz")
    n = 28
    if n > qb.qubit_cap():
        qb.set_qubit_cap(n)
    circ = bench_circuit(n, 1, g["theta"])
    reg = qb.zero_state(n)
    qb.apply(reg, circ)
    e = qb.expect(qb.heisenberg(n), reg)
    assert vec_err(e, g["energy"]) <= TOL
    idx = g["probe_idx"]
    # probe amplitudes without downloading the 4 GiB state: 16-byte reads of the device buffer (B = 1)
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12")
    qb.synchronize()
    got = np.empty(len(idx), dtype=np.complex128)
    for k, i in enumerate(idx):
        rc = cudart.cudaMemcpy(ctypes.c_void_p(got.ctypes.data + 16 * k), ctypes.c_void_p(reg.device_ptr + 16 * int(i)),
                               ctypes.c_size_t(16), 2)  # cudaMemcpyDeviceToHost
        assert rc == 0
    assert amp_err(got, g["probes"]) <= TOL
