"""SURVEY §8(d) cfg 3 on one B200: QCBM-style batched reverse-mode AD.

  energy: 1000 product states (bitstrings Rng(42).bits() & (2^20-1), batch innermost),
          variational_circuit(20, 10), loss Σ_b <ψ_b|heisenberg(20)|ψ_b>, gradient summed over b
  mmd   : B = 1, target_p = normalize(U(0,1)^{2^20}) from Rng(42), brbf_kernel(2.0), reverse mode

Device-timed with CUDA events (steady state, after a warm-up step that also JIT-compiles).
Gates/s counts forward + backward gates (2G per state per step)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--depth", type=int, default=10)
    ap.add_argument("--batch", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dtype", default="c128")
    a = ap.parse_args()
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    n, d, Bn = a.n, a.depth, a.batch
    circ = qb.variational_circuit(n, d)
    qb.dispatch(circ, "random", rng=qb.Rng(42))
    G = n * (1 + 4 * d)
    h = qb.heisenberg(n)
    rng = qb.Rng(42)
    bits = [rng.bits() & ((1 << n) - 1) for _ in range(Bn)]
    reg = qb.product_state(bits, n, nbatch=Bn, dtype=a.dtype)
    ms, res = timed(lambda: qb.expect_grad(h, (reg, circ), inplace=True), a.reps)
    S = (16 if a.dtype == "c128" else 8) << n
    out = [{"cfg": "3-energy", "n": n, "depth": d, "batch": Bn, "dtype": a.dtype, "ms_per_step": ms,
            "gates_per_s": 2 * G * Bn / (ms / 1e3), "state_GB": S * Bn / 1e9,
            "loss": float(np.sum(res.energies)), "grad_norm": float(np.linalg.norm(res.param_grads)),
            "passes": qb.compile_block(circ).stats()}]
    # MMD variant: B = 1
    r2 = qb.Rng(42)
    q = np.fromiter((r2.uniform() for _ in range(1 << n)), dtype=np.float64, count=1 << n)
    q /= q.sum()
    mmd = qb.MMD(qb.brbf_kernel(2.0), q)
    reg1 = qb.zero_state(n, dtype=a.dtype)
    ms2, res2 = timed(lambda: qb.expect_grad(mmd, (reg1, circ), inplace=True), max(3, a.reps))
    adj = qb.Register(n, 1, dtype=a.dtype)
    ms3, _ = timed(lambda: qb.mmd_seed(mmd, reg1, adj), 10)
    out.append({"cfg": "3-mmd", "n": n, "depth": d, "batch": 1, "dtype": a.dtype, "ms_per_step": ms2,
                "gates_per_s": 2 * G / (ms2 / 1e3), "mmd": float(res2.energies[0]), "band": mmd.band,
                "seed_ms": ms3, "grad_norm": float(np.linalg.norm(res2.param_grads))})
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
