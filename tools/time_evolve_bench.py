"""Device Krylov time evolution at the metric size: e^{-iHt}|ψ> for heisenberg(n), device-timed.
    python tools/time_evolve_bench.py [--n 25]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=25)
    a = ap.parse_args()
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    h = qb.heisenberg(a.n)
    reg = qb.rand_state(a.n, 1, seed=42)
    e0 = float(qb.expect(h, reg)[0])
    qb.evolve(reg, h, 0.01)  # warm-up (JIT of the seed passes, buffers)
    for t in (0.1, 1.0):
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        k = qb.evolve(reg, h, t)
        ev1.record()
        torch.cuda.synchronize()
        print(json.dumps({"n": a.n, "t": t, "krylov_dim": k, "ms": ev0.elapsed_time(ev1),
                          "energy_drift": abs(float(qb.expect(h, reg)[0]) - e0), "norm": float(reg.norm(0))}),
              flush=True)


if __name__ == "__main__":
    main()
