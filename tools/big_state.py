"""Large states on one B200 (SURVEY §8(d) cfg 5 building blocks).

  single : variational_circuit(n, depth) forward + <heisenberg(n)> + <Σ Z_i> on one register
           (n = 33 is 128 GiB complex128: the per-GPU share of the 36-qubit / 8-GPU state)
  sharded: the same circuit over 2^g virtual ranks (DeviceVirtualBackend) with qubit-swap
           exchanges, checked against the single-register energies at a size where both fit

    python tools/big_state.py --n 33 --depth 2 [--sharded-g 3 --check-n 30]
"""
import argparse
import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_10877_b200 as qb  # noqa: E402
from paper_1912_10877_b200 import blocks as B  # noqa: E402
from paper_1912_10877_b200._capi import check, lib  # noqa: E402
from paper_1912_10877_b200.sharded import DeviceVirtualBackend, ShardedState  # noqa: E402


def events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def zsum(n):
    return qb.Add([qb.put(n, q, qb.Z) for q in range(1, n + 1)])


def single(n, depth, seed=42):
    qb.set_qubit_cap(max(n, 30))
    circ = qb.variational_circuit(n, depth)
    qb.dispatch(circ, "random", rng=qb.Rng(seed))
    reg = qb.zero_state(n)
    qb.compile_block(circ)
    e0, e1 = events()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    qb.apply(reg, circ)
    e1.record()
    torch.cuda.synchronize()
    ms_apply = e0.elapsed_time(e1)
    wall = time.perf_counter() - t0
    e0.record()
    eh = float(qb.expect(qb.heisenberg(n), reg)[0])
    ez = float(qb.expect(zsum(n), reg)[0])
    e1.record()
    torch.cuda.synchronize()
    G = n * (1 + 4 * depth)
    out = {"mode": "single", "n": n, "depth": depth, "gates": G, "apply_ms": ms_apply, "apply_wall_s_incl_jit": wall,
           "gates_per_s": G / (ms_apply / 1e3), "expect_ms": e0.elapsed_time(e1), "E_heisenberg": eh, "E_zsum": ez,
           "norm": float(reg.norm(0)), "state_GiB": (16 << n) / 2**30, "passes": qb.compile_block(circ).stats()}
    del reg
    gc.collect()
    torch.cuda.synchronize()
    return out


def sharded(n, depth, g, seed=42, staging=2 << 30):
    """The same circuit over 2^g virtual ranks on this GPU: the chunked remaps (libqbg pack /
    unpack kernels through the staging arena) timed with CUDA events; second run = steady state."""
    circ = qb.variational_circuit(n, depth)
    qb.dispatch(circ, "random", rng=qb.Rng(seed))
    be = DeviceVirtualBackend(n, g, staging_bytes=staging)
    st = ShardedState(be, n, g)
    remaps = []
    orig = be.remap

    def timed_remap(pairs):
        a, b = events()
        a.record()
        orig(pairs)
        b.record()
        torch.cuda.synchronize()
        remaps.append((len(pairs), a.elapsed_time(b)))

    be.remap = timed_remap
    out = None
    for rep in range(2):
        st.reset_zero()
        remaps.clear()
        moved0 = be.bytes_moved
        e0, e1 = events()
        torch.cuda.synchronize()
        e0.record()
        st.apply(circ)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        eh = st.expect_pauli(B.pauli_terms(qb.heisenberg(n)))
        ez = st.expect_pauli(B.pauli_terms(zsum(n)))
        moved = be.bytes_moved - moved0
        rms = sum(t for _, t in remaps)
        out = {"mode": "sharded-virtual", "n": n, "g": g, "depth": depth, "run": rep,
               "apply_ms" + ("_incl_jit" if rep == 0 else ""): ms, "E_heisenberg": eh, "E_zsum": ez,
               "remaps": len(remaps), "qubit_moves": sum(j for j, _ in remaps), "remap_ms_total": rms,
               "bytes_moved_all_ranks": moved,
               "remap_gbs": moved / (rms / 1e3) / 1e9 if rms else None,
               "note": "virtual ranks on one GPU: every moved byte is packed and unpacked in HBM (4 x traffic)"}
    del st, be
    gc.collect()
    torch.cuda.synchronize()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=33)
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--sharded-g", type=int, default=3)
    ap.add_argument("--check-n", type=int, default=28)
    a = ap.parse_args()
    check(lib().qbg_set_stream(torch.cuda.current_stream().cuda_stream))
    res = [single(a.check_n, a.depth), sharded(a.check_n, a.depth, a.sharded_g)]
    res[1]["matches_single"] = abs(res[1]["E_heisenberg"] - res[0]["E_heisenberg"]) < 1e-9 and \
        abs(res[1]["E_zsum"] - res[0]["E_zsum"]) < 1e-9
    res.append(single(a.n, a.depth))
    res.append(single(a.n, a.depth))  # second run: JIT cached, steady state
    res.append(sharded(a.n, a.depth, a.sharded_g))
    res[-1]["matches_single"] = abs(res[-1]["E_heisenberg"] - res[-2]["E_heisenberg"]) < 1e-9
    for r in res:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
