"""Runs a few apply+grad steps of the bench workload (for ncu / compute-sanitizer captures).

    python tools/profile_step.py [--qubits 25] [--depth 10] [--steps 2] [--no-fusion]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1912_10877_b200 as qb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=25)
    ap.add_argument("--depth", type=int, default=10)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-fusion", action="store_true")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    a = ap.parse_args()
    qb.set_fusion(not a.no_fusion)
    if a.qubits > qb.qubit_cap():
        qb.set_qubit_cap(a.qubits)
    circ = qb.variational_circuit(a.qubits, a.depth)
    qb.dispatch(circ, "random")
    h = qb.heisenberg(a.qubits)
    reg = qb.zero_state(a.qubits, a.batch, dtype=a.dtype)
    for _ in range(a.steps):
        t0 = time.perf_counter()
        r = qb.expect_grad(h, (reg, circ))
        qb.synchronize()
        print(f"step {(time.perf_counter() - t0) * 1e3:.2f} ms E={r.energies[0]:.12f}", flush=True)
    print(qb.compile_block(circ).stats())


if __name__ == "__main__":
    main()
