"""Host-side cost of one optimiser step of the bench workload (25q/d10 expect'): the device-timed
step vs the same step with a new θ every time (dispatch + values-only plan refresh) vs the bench's
e2e loop (new θ + zero_state + result read-back).  Wall-clock per step, after warm-up.

    python tools/e2e_breakdown.py [--steps 10]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    L = lib()
    check(L.qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    n, d = 25, 10
    circ = qb.variational_circuit(n, d)
    qb.dispatch(circ, "random", rng=qb.Rng(42))
    h = qb.heisenberg(n)
    reg = qb.zero_state(n)
    theta = qb.parameters(circ)
    for _ in range(3):
        qb.expect_grad(h, (reg, circ))
    torch.cuda.synchronize()

    def timed(fn):
        t0 = time.perf_counter()
        for _ in range(a.steps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / a.steps

    same = timed(lambda: qb.expect_grad(h, (reg, circ)))
    th = theta.copy()

    def new_theta():
        th[:] += 1e-9
        qb.dispatch(circ, th)
        qb.expect_grad(h, (reg, circ))

    newt = timed(new_theta)
    p = qb.compile_block(circ)

    def sync_only():
        th[:] += 1e-9
        qb.dispatch(circ, th)
        p.sync_params()

    t_sync = timed(sync_only)

    def disp_only():
        th[:] += 1e-9
        qb.dispatch(circ, th)

    t_disp = timed(disp_only)
    print(f"step, same θ: {same:.3f} ms; step, new θ: {newt:.3f} ms (+{newt - same:.3f}); "
          f"dispatch alone {t_disp:.3f} ms; dispatch + parameter sync (plan refresh is lazy) {t_sync:.3f} ms")


if __name__ == "__main__":
    main()
