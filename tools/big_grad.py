"""Largest single-GPU gradients: expect' in place (ψ and φ̄ only, 2 x 2^n x 16 B) at n = 32
(128 GiB), and the out-of-memory path at n = 33 (must raise ResourceError, not crash)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402


def main():
    qb.set_qubit_cap(34)
    n = int(os.environ.get("N", 32))
    circ = qb.variational_circuit(n, 1)
    qb.dispatch(circ, "random", rng=qb.Rng(42))
    h = qb.heisenberg(n)
    reg = qb.zero_state(n)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = qb.expect_grad(h, (reg, circ), inplace=True)
        torch.cuda.synchronize()
        print(json.dumps({"n": n, "depth": 1, "inplace": True, "rep": rep, "seconds": time.perf_counter() - t0,
                          "energy": float(r.energies[0]), "grad_norm": float((r.param_grads ** 2).sum() ** 0.5),
                          "state_GiB": (16 << n) / 2 ** 30}), flush=True)
    try:
        qb.expect_grad(h, (reg, circ), inplace=False)  # needs a third state
        print(json.dumps({"n": n, "inplace": False, "result": "fit"}))
    except qb.errors.ResourceError as e:
        print(json.dumps({"n": n, "inplace": False, "result": "ResourceError", "msg": str(e)[:120]}))


if __name__ == "__main__":
    main()
