"""SURVEY §8(d) cfg 4: 30-qubit variational circuits (16 GiB complex128 state), forward apply,
fused tile passes vs one kernel per gate, device-timed; plus apply+grad (fused)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = int(os.environ.get("N", 30))
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    reg = qb.zero_state(n)
    h = qb.heisenberg(n)
    for d in (1, 2, 10):
        circ = qb.variational_circuit(n, d)
        qb.dispatch(circ, "random", rng=qb.Rng(42))
        G = n * (1 + 4 * d)
        out = {"cfg": "4", "n": n, "depth": d, "gates": G}
        for fused in (True, False):
            qb.set_fusion(fused)
            ms = timed(lambda: qb.apply(reg, circ))
            out["fused_apply_ms" if fused else "pergate_apply_ms"] = ms
        qb.set_fusion(True)
        out["fused_gates_per_s"] = G / (out["fused_apply_ms"] / 1e3)
        out["pergate_gates_per_s"] = G / (out["pergate_apply_ms"] / 1e3)
        out["speedup_fused_vs_pergate"] = out["pergate_apply_ms"] / out["fused_apply_ms"]
        out["passes"] = qb.compile_block(circ).stats()
        if d == 10:
            out["apply_grad_ms"] = timed(lambda: qb.expect_grad(h, (reg, circ), inplace=True), 1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
