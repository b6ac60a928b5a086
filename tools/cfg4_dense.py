"""BASELINE cfg 4 A/B: variational_circuit(n, d) forward on one B200, three ways —
  tile : the default tile engine (fused.cu: 2x2 / 4x4 gate runs inside shared-memory tiles);
  dense: gate fusion into dense 5-qubit blocks (densefuse.py), each block one HBM pass on the tensor
         cores — DMMA m8n8k4 in complex128 (dense_mma.cu), tcgen05 kind::tf32 with a 3-piece split
         in complex64 (dense_tc.cu);
  cuda : the same dense blocks on the CUDA-core per-gate kernel;
  tf32 : (complex64) the dense blocks on tcgen05 kind::tf32 with a 3-piece split.
Prints one JSON line per mode (device-timed, median of --reps) and checks the dense-block state
against the tile engine's (<ψ_tile|ψ_dense> = 1 and equal energies).

    python tools/cfg4_dense.py --n 30 --depth 10 [--modes tile,dense] [--reps 3] [--dtype c64]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402
from paper_1912_10877_b200.densefuse import fuse_dense  # noqa: E402


def timed(fn, reps):
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(torch.cuda.current_stream())
        fn()
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


def profile(fn):
    import ctypes
    L = lib()
    L.qbg_profile_reset()
    L.qbg_profile_enable(1)
    fn()
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    check(L.qbg_profile_report(buf, len(buf)))
    L.qbg_profile_enable(0)
    out = {}
    for line in buf.value.decode().strip().splitlines():
        name, cnt, tot, byt, flo = line.split("\t")
        out[name] = {"launches": int(cnt), "ms": float(tot), "GB/s": float(byt) / (float(tot) / 1e3) / 1e9 if float(tot) else 0,
                     "TFLOP/s": float(flo) / (float(tot) / 1e3) / 1e12 if float(tot) else 0}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--depth", type=int, default=10)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--modes", default="tile,dense")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dtype", default="c128")
    args = ap.parse_args()
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    n, d = args.n, args.depth
    if n > qb.qubit_cap():
        qb.set_qubit_cap(n)
    circ = qb.variational_circuit(n, d)
    qb.dispatch(circ, "random", rng=qb.Rng(42))
    G = n * (1 + 4 * d)
    h = qb.heisenberg(n)
    t0 = time.perf_counter()
    dense = fuse_dense(circ, args.k)
    plan_s = time.perf_counter() - t0
    S = (16 if args.dtype == "c128" else 8) << n
    ref = None
    for mode in args.modes.split(","):
        qb.set_fusion(mode == "tile")
        qb.set_dense_path({"cuda": "cuda", "tf32": "tf32-tensor"}.get(mode, "fp64-tensor"))
        blk = circ if mode == "tile" else dense
        reg = qb.zero_state(n, dtype=args.dtype)
        qb.apply(reg, blk)  # warm-up: plans, kernels
        torch.cuda.synchronize()

        def run():
            check(lib().qbg_set_zero(reg._h))
            qb.apply(reg, blk)

        ms = timed(run, args.reps)
        prof = profile(run)
        e = float(qb.expect(h, reg)[0])
        line = {"mode": mode, "n": n, "depth": d, "dtype": args.dtype, "gates": G, "forward_ms": ms,
                "gates_per_s": G / (ms / 1e3), "energy": e, "kernels": prof,
                "hbm_passes": sum(v["launches"] for k, v in prof.items() if k in ("fused_fwd", "dense_mma", "dense_tc", "gate")),
                "dense_blocks": len(dense.blocks) if mode != "tile" else None,
                "host_fusion_s": plan_s if mode != "tile" else None,
                "per_gate_roofline_ms": 2 * G * S / 6553.3e9 * 1e3}
        if ref is None:
            ref = (mode, reg, e)
        else:
            ip = reg.inner(ref[1])[0]
            line["check_vs_" + ref[0]] = {"abs_inner_minus_1": abs(abs(ip) - 1.0), "energy_diff": abs(e - ref[2])}
            del reg
        print(json.dumps(line), flush=True)
    qb.set_fusion(True)
    qb.set_dense_path("fp64-tensor")


if __name__ == "__main__":
    main()
