"""Small-n workload for compute-sanitizer (memcheck / racecheck / synccheck): fused forward +
expect' (JIT pipelined passes, seed, reverse, epilogue), per-gate kernels, MMD, Krylov."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200 import blocks as B  # noqa: E402


def main():
    n = 12
    circ = qb.variational_circuit(n, 2)
    qb.dispatch(circ, "random")
    h = qb.heisenberg(n)
    reg = qb.rand_state(n, 2, seed=1)
    r = qb.expect_grad(h, (reg, circ))
    qb.dispatch(circ, qb.parameters(circ) + 0.1)  # new θ: values-only plan refresh
    r = qb.expect_grad(h, (reg, circ))
    qb.set_fusion(False)
    r2 = qb.expect_grad(h, (reg, circ))
    qb.set_fusion(True)
    assert np.abs(r.param_grads - r2.param_grads).max() < 1e-10
    q = np.full(1 << n, 1.0 / (1 << n))
    qb.expect_grad(qb.MMD(qb.brbf_kernel(2.0), q), (qb.zero_state(n), circ))
    r1 = qb.zero_state(n)
    qb.evolve(r1, h, 0.2)
    qb.measure(r1, 100)
    print("sanitize smoke ok", float(r.energies[0]))


if __name__ == "__main__":
    main()
