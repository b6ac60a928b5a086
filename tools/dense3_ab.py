"""3-qubit dense gates fused into tile passes (OP_DENSE3) vs one DMMA pass per gate: layers of
random 3-qubit unitaries + rotation layers at 25 qubits, forward, device-timed.

    python tools/dense3_ab.py [--n 25] [--layers 6]
    QBG_TILE_DENSE3=0 python tools/dense3_ab.py      # the planner without the stage op (A/B)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200 import blocks as B  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=25)
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--t", type=int, default=3, help="qubits per dense block (3 or 4)")
    a = ap.parse_args()
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    rng = np.random.default_rng(1)
    n = a.n
    blocks = []
    for layer in range(a.layers):
        t = a.t
        off = layer % t
        for s in range(off, n - t + 1, t):
            z = rng.normal(size=(1 << t, 1 << t)) + 1j * rng.normal(size=(1 << t, 1 << t))
            blocks.append(B.put(n, tuple(range(s + 1, s + t + 1)), B.matblock(np.linalg.qr(z)[0])))
        for q in range(1, n + 1):
            blocks.append(B.put(n, q, B.Rx(float(rng.uniform(0, 6.28)))))
    circ = B.chain(n, *blocks)
    ndense = sum(1 for b in blocks if len(b.locs) == a.t)
    res = {}
    states = {}
    for mode in ("fused", "per-gate"):
        qb.set_fusion(mode == "fused")
        reg = qb.zero_state(n)
        qb.apply(reg, circ)
        torch.cuda.synchronize()
        ms = []
        for _ in range(3):
            check(lib().qbg_set_zero(reg._h))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            qb.apply(reg, circ)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        res[mode] = {"forward_ms": float(np.median(ms)), "stats": qb.compile_block(circ).stats()}
        states[mode] = reg
    qb.set_fusion(True)
    ip = states["fused"].inner(states["per-gate"])[0]
    print(json.dumps({"tile_dense3": os.environ.get("QBG_TILE_DENSE3", "1"), "n": n, "layers": a.layers, "t": a.t, "dense_gates": ndense, "rotations": len(blocks) - ndense, **res,
                      "speedup": res["per-gate"]["forward_ms"] / res["fused"]["forward_ms"],
                      "abs_inner_minus_1": abs(abs(ip) - 1.0)}))


if __name__ == "__main__":
    main()
