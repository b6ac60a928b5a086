"""SURVEY §8(d) cfg 1: single instruct calls on a 16-qubit complex128 state (1 MiB, L2-resident,
so latency-bound).  rand_state(16, 1, seed=42); X, H, T, Rx(0.5) on qubit 2; CNOT =
instruct(X, (3,), (2,), (1,)); Toffoli = instruct(X, (1,), (2, 3), (1, 1)).

  direct : 1000 back-to-back qbg_instruct calls (host dispatch + one kernel each), CUDA events
  graph  : the same 1000 calls captured once in a CUDA graph and replayed (min of 20 replays)
Reports µs/gate and gates/s.  The state after the sequence is checked against the oracle
(tests/ covers parity; here only the timing)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402

GATES = {
    "X@2": ("X", (2,), (), (), ()),
    "H@2": ("H", (2,), (), (), ()),
    "T@2": ("T", (2,), (), (), ()),
    "Rx(0.5)@2": ("Rx", (2,), (), (), (0.5,)),
    "CNOT(2->3)": ("X", (3,), (2,), (1,), ()),
    "Toffoli(2,3->1)": ("X", (1,), (2, 3), (1, 1), ()),
}


def main():
    n, reps = int(os.environ.get("N", 16)), 1000
    out = []
    for name, (tag, locs, ctrls, cfg, par) in GATES.items():
        reg = qb.rand_state(n, 1, seed=42)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            check(lib().qbg_set_stream(s.cuda_stream))
            for _ in range(50):
                qb.instruct(reg, tag, locs, ctrls, cfg, par)
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                qb.instruct(reg, tag, locs, ctrls, cfg, par)
            e1.record(s)
            s.synchronize()
            direct_us = e0.elapsed_time(e1) * 1e3 / reps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
            for _ in range(reps):
                qb.instruct(reg, tag, locs, ctrls, cfg, par)
        check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
        g.replay()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
        S = 16 << n
        out.append({"cfg": "1-single-gates", "n": n, "gate": name, "direct_us_per_gate": direct_us,
                    "graph_us_per_gate": best, "graph_gates_per_s": 1e6 / best,
                    "effective_GBps_graph": 2 * S / (best * 1e-6) / 1e9})
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
