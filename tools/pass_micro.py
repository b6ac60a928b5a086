"""Micro-benchmarks of single fused passes at 25 qubits (device-timed with CUDA events).

Isolates the memory behaviour of the tile machinery from the FP64 work:
  diag     : 25 Rz gates            -> one pass, diagonal ops only (no register targets)
  dense1   : one Rx on qubit 14     -> one pass, one stage, one dense op
  stages   : Rx on 12 qubits        -> one pass, several stages (transposes)
  copy     : torch copy of the state (reference for the HBM roofline)
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
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
    n = 25
    S = 16 << n
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    reg = qb.rand_state(n)
    cases = {
        "diag": qb.chain(n, *[qb.put(n, q, qb.Rz(0.1 * q)) for q in range(1, n + 1)]),
        "dense1": qb.chain(n, qb.put(n, 14, qb.Rx(0.3))),
        "stages": qb.chain(n, *[qb.put(n, q, qb.Rx(0.1 * q)) for q in range(4, 13)]),
        "stages_low": qb.chain(n, *[qb.put(n, q, qb.Rx(0.1 * q)) for q in range(1, 10)]),
    }
    for name, c in cases.items():
        p = qb.compile_block(c)
        ms = timeit(lambda: qb.apply(reg, c))
        info = [l for l in p.plan_info().splitlines() if "tile" in l]
        print(f"{name:10s} {ms * 1e3:8.1f} us  {2 * S / (ms * 1e-3) / 1e9:7.0f} GB/s  passes={len(info)}  {info[:1]}")
    x = torch.empty(S // 8, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ms = timeit(lambda: y.copy_(x))
    print(f"{'copy':10s} {ms * 1e3:8.1f} us  {2 * S / (ms * 1e-3) / 1e9:7.0f} GB/s")


if __name__ == "__main__":
    main()
