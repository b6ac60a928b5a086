#!/usr/bin/env python
"""Headline benchmark: gates/s (and HBM GB/s) of the 25-qubit variational circuit
apply + reverse-AD gradient (BASELINE.json metric, config[1] as the metric run:
``expect'(heisenberg(25), zero_state(25) => variational_circuit(25, 10))``, complex128).

One step = one expect_grad: forward G gates, seed φ̄ = Oψ (T Pauli terms), backward G gates
(uncompute + gradient).  value = N·2G / t_step (weak scaling: each rank runs one replica with
its own parameters — the 25-qubit problem fits one B200, so multi-GPU is replicas only).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gates/sec & HBM GB/s, 25-qubit variational circuit apply+grad, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--qubits", type=int, default=25)
    ap.add_argument("--depth", type=int, default=10)
    ap.add_argument("--no-fusion", action="store_true")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"],
                    help="register precision (the metric is quoted in c128; c64 is reported beside it)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU sample for cpu_baseline")
    ap.add_argument("--no-sharded", action="store_true", help="skip the sharded-state weak-scaling measurement")
    ap.add_argument("--sharded-local-qubits", type=int, default=33,
                    help="qubits per GPU of the sharded state (33: 128 GiB per B200; n = this + log2 N)")
    ap.add_argument("--sharded-depth", type=int, default=2)
    ap.add_argument("--sharded-steps", type=int, default=3)
    ap.add_argument("--sharded-timeout", type=float, default=420.0,
                    help="seconds after which a stuck sharded measurement is reported as an error")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---- clocks sampler (B200_PROFILING.md "clocks DURING the timed region") -------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, local_rank: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        self.idx = vis.split(",")[local_rank] if vis else str(local_rank)
        self.proc = None
        self.path = None
        self.skip = 0

    def start(self):
        """Start sampling every 20 ms and return once the sampler has produced its first line, so
        the timed region that follows is covered from its first step."""
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            import shutil
            pre = ["stdbuf", "-oL"] if shutil.which("stdbuf") else []  # line-buffered into the file
            self.proc = subprocess.Popen(
                pre + ["nvidia-smi", "-i", self.idx, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 10.0 and self.proc.poll() is None:
                if os.path.getsize(self.path) > 0:
                    break
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def mark(self):
        """Line count at the start of the timed region: samples before it are not reported."""
        if self.proc is None:
            return
        with open(self.path) as f:
            self.skip = sum(1 for _ in f)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for i, line in enumerate(open(self.path)):
            if i < self.skip:
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        # the sampler runs across the whole timed region; report the median of loaded samples
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- reference arm: the reference's CPU implementation on the host cores --------------------------
def cpu_validation():
    """The bounded CPU sample's extrapolation checked against full timed reference runs
    (profiles/r02/cpu_baseline_validation.json: 20q and 25q apply+grad, one core)."""
    try:
        v = json.load(open(os.path.join(ROOT, "profiles", "r02", "cpu_baseline_validation.json")))
        return {k: round(x["ratio_extrap_over_full"], 3) for k, x in v.items()} | {
            "note": "extrapolated job time / full timed reference run: < 1 means the reported reference rate is "
                    "optimistic (the reference is slower than stated)"}
    except Exception:
        return None


def run_reference(args, rank, world):
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_baseline as cb
    import oracle as O
    orc = O.reference()
    kind = "reference"
    if orc is None:
        orc, kind = O.restatement(), "port"
    threads = cb.nproc()
    steps = args.steps + args.warmup
    # size each step so the whole run stays within ~3 minutes: ~2-3 s per (k=1, m=1) sample
    k, m = (2, 3) if steps <= 12 else (1, 1)
    vals, samples = [], None
    for s in range(steps):
        r = cb.sample_apply_grad(orc, args.qubits, args.depth, k, m, threads=threads)
        samples = r
        if s >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    ms = 2 * args.qubits * (1 + 4 * args.depth) / v * 1e3
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": "gates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": "gates/s", "cores": threads, "kind": kind,
                         "sample": samples["sample"] + f"; {threads} threads requested (the reference parallelises "
                                                       "over register columns only, so an unbatched state runs on "
                                                       "1 core, utils.hpp:37-64)",
                         "cpu_model": cb.cpu_model(), "extrapolation_check": cpu_validation()},
        "e2e": {"value": v, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def fp64_roofline(top, per_launch_ms):
    """The tile passes are FP64-bound as much as HBM-bound: the same kernel's
    algorithmic FP64 work (pass_flops in fused.cu) against the measured DFMA peak."""
    if not top or not top.get("flops"):
        return None
    peak, src = 37.0, "nominal 64 DFMA/clk/SM x 148 SMs x 1.965 GHz"
    try:
        peak = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_pipes.json")))["dfma_tflops"]
        src = "measured DFMA peak (profiles/r01_fp64_pipes.json, tools/fp64_pipes.cu)"
    except Exception:
        pass
    ach = top["flops"] / top["launches"] / (per_launch_ms / 1e3) / 1e12
    return {"achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "flops_per_launch": top["flops"] / top["launches"], "peak_source": src}


def per_gate_roofline(top, per_launch_ms, G, S, peak):
    """SURVEY §8(d)'s algorithmic unit: one gate on one state = 2S bytes, a reverse-pass gate = 2
    units.  The fused launches of a step together apply every gate once, so one launch of the
    dominant kernel stands for (gates x bytes per gate) / (its launches per step); above 1.0 means
    fusion beat the per-gate roofline."""
    if not top or top["name"] not in ("fused_bwd", "fused_fwd"):
        return None
    per_gate = (4 if top["name"] == "fused_bwd" else 2) * S
    bpl = G * per_gate / (top["launches"] / 2)
    ach = bpl / (per_launch_ms / 1e3) / 1e9
    return {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "bytes_per_launch": bpl,
            "unit_definition": "2S per gate per state pass (forward 2S, reverse 4S), SURVEY 8(d)"}


def workload_config(args):
    n, d = args.qubits, args.depth
    G, P, T = n * (1 + 4 * d), n * (1 + 3 * d), 3 * (n - 1)
    cplx = "complex128" if args.dtype == "c128" else "complex64"
    return {"workload": f"expect'(heisenberg({n}) open, zero_state({n}) => variational_circuit({n},{d})) "
                        f"apply+grad, {cplx}",
            "qubits": n, "depth": d, "gates_fwd": G, "gates_per_step": 2 * G, "params": P, "terms": T,
            "batch": 1, "state_bytes": (16 if args.dtype == "c128" else 8) << n,
            "l2": f"state {(16 if args.dtype == 'c128' else 8) << n >> 20} MiB > 126 MB L2: inputs larger than L2, "
                  "no flush",
            "parallelism": f"replicas x{args.gpus}"}


# ---- sharded states: SURVEY §8(e) / BASELINE cfg 5, weak scaling 33q/1, 34q/2, 35q/4, 36q/8 ------------
def sharded_weak_scaling(args, rank, world, pg):
    """variational_circuit(n, depth) forward + <heisenberg(n)> on one n-qubit state split over the N
    GPUs (n = local + log2 N; each GPU holds a 2^local complex128 shard), global qubits moved by
    the chunked all-to-all remaps of sharded.py over NCCL.  Device-timed (CUDA events on the
    library stream), max over ranks.  gates/s counts the circuit's gates on the whole state."""
    import torch
    import paper_1912_10877_b200 as qb
    from paper_1912_10877_b200.sharded import DeviceNcclBackend, ShardedState
    g = world.bit_length() - 1
    if world != 1 << g:
        return {"skipped": "world size is not a power of two"}
    nl, d = args.sharded_local_qubits, args.sharded_depth
    n = nl + g
    # every rank must fit its shard + the staging arena + headroom, or none starts: a rank that
    # failed alone would leave the others waiting in NCCL
    free, _ = torch.cuda.mem_get_info()
    need = (16 << nl) + (2 << 30) + (4 << 30)
    ok = torch.tensor([1.0 if free >= need else 0.0], device="cuda")
    if pg is not None:
        pg.all_reduce(ok, op=pg.ReduceOp.MIN)
    if float(ok.item()) < 1.0:
        return {"skipped": f"a rank has {free / 2**30:.1f} GiB free < {need / 2**30:.1f} GiB (shard + staging + headroom)"}
    if n > qb.qubit_cap():
        qb.set_qubit_cap(n)
    circ = qb.variational_circuit(n, d)
    qb.dispatch(circ, "random", rng=qb.Rng(42))
    h = qb.heisenberg(n)
    terms = qb.pauli_terms(h)
    be = DeviceNcclBackend(n, g)
    st = ShardedState(be, n, g)
    stream = torch.cuda.current_stream()

    def barrier():
        if pg is not None:
            pg.barrier()

    def one():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        st.reset_zero()
        e[0].record(stream)
        st.apply(circ)
        e[1].record(stream)
        energy = st.expect_pauli(terms)
        e[2].record(stream)
        return e, energy

    one()  # warm-up: segment programs, kernels, staging arena
    torch.cuda.synchronize()
    barrier()
    ex0_b = be.exchange.bytes_sent
    be.exchange.events = []
    apply_ms, exp_ms, energy = [], [], None
    for _ in range(args.sharded_steps):
        e, energy = one()
        torch.cuda.synchronize()
        apply_ms.append(e[0].elapsed_time(e[1]))
        exp_ms.append(e[1].elapsed_time(e[2]))
    barrier()
    a, x = statistics.median(apply_ms), statistics.median(exp_ms)
    if pg is not None:
        t = torch.tensor([a, x], device="cuda")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        a, x = float(t[0]), float(t[1])
    G = n * (1 + 4 * d)
    S_local = 16 << nl
    remaps = [len(p) for p in st.sched.exchanges]
    per_step_bytes = (be.exchange.bytes_sent - ex0_b) / max(1, args.sharded_steps)
    out = {"workload": f"variational_circuit({n},{d}) forward + <heisenberg({n})> open, complex128, "
                       f"{world} GPU(s) x 2^{nl} amplitudes", "qubits": n, "local_qubits": nl, "global_qubits": g,
           "gates": G, "apply_ms": a, "expect_ms": x, "step_ms": a + x, "gates_per_s": G / (a / 1e3),
           "energy": energy, "scaling": "weak",
           "hbm_gbs_alg_per_gpu": G * 2 * S_local / (a / 1e3) / 1e9,
           "exchange_bytes_per_step_per_gpu": per_step_bytes,
           "exchanges_per_step": len(remaps) // (args.sharded_steps + 1) if remaps else 0,
           "staging_bytes": be.exchange.staging_bytes,
           "memory_note": "per GPU: shard (16 x 2^local B) + staging arena; the tile engine's plan tables"}
    if be.exchange.events:
        # pack + NCCL send/recv + unpack of every remap (device-timed on the library stream)
        ex_ms = sum(e0.elapsed_time(e1) for e0, e1 in be.exchange.events) / args.sharded_steps
        if pg is not None:
            t = torch.tensor([ex_ms], device="cuda")
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            ex_ms = float(t[0])
        out["exchange_ms_per_step"] = ex_ms
        out["nvlink_gbs_per_gpu"] = per_step_bytes / (ex_ms / 1e3) / 1e9  # bytes sent per direction
    del st, be
    return out


# ---- our arm ------------------------------------------------------------------------------------
def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        from datetime import timedelta
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=timedelta(minutes=10))
        pg = dist

    import paper_1912_10877_b200 as qb
    from paper_1912_10877_b200._capi import check, lib
    L = lib()
    check(L.qbg_set_device(local))
    stream = torch.cuda.current_stream()
    check(L.qbg_set_stream(stream.cuda_stream))
    qb.set_fusion(not args.no_fusion)
    if args.qubits > qb.qubit_cap():
        qb.set_qubit_cap(args.qubits)

    n, d = args.qubits, args.depth
    circ = qb.variational_circuit(n, d)
    qb.dispatch(circ, "random", rng=qb.Rng(42 + rank))
    h = qb.heisenberg(n)
    G, T = n * (1 + 4 * d), 3 * (n - 1)
    S = (16 if args.dtype == "c128" else 8) << n
    reg = qb.zero_state(n, dtype=args.dtype)
    prog = qb.compile_block(circ)
    qb.compile_observable(h)

    def barrier():
        if pg is not None:
            pg.barrier()

    def step():
        return qb.expect_grad(h, (reg, circ))

    for _ in range(max(3, args.warmup)):
        res = step()
    torch.cuda.synchronize()

    # ---- timed region (device events on the library's stream) ----
    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    torch.cuda.synchronize()
    clocks.mark()
    L.qbg_launch_count_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = int(L.qbg_launch_count())
    barrier()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if pg is not None:
        t = torch.tensor([ms], device="cuda")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    value = world * 2 * G / (ms / 1e3)
    alg_bytes = (6 * G + 3 * T + 2) * S
    hbm_alg = alg_bytes / (ms / 1e3) / 1e9

    # ---- end to end through the public API: host θ in (pinned), host energies/grads out ----
    theta = qb.parameters(circ)
    th_pin = torch.from_numpy(theta).pin_memory()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.steps):
        th_pin.add_(1e-9)  # a VQE-style update each step so the parameters really cross
        qb.dispatch(circ, th_pin.numpy())
        check(L.qbg_set_zero(reg._h))
        r2 = step()
        _ = (float(r2.energies[0]), r2.param_grads.sum())
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if pg is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": world * 2 * G / (e2e_ms / 1e3), "unit": "gates/s", "h2d_bytes_per_step": 8 * theta.size,
           "d2h_bytes_per_step": 8 * theta.size + 8,
           "path": "dispatch(θ from pinned host) + zero_state + expect' + energies/grads to host, per step"}

    # variant: input state uploaded from pinned host memory every step (qbg_upload)
    host_state = torch.zeros(2 << n, dtype=torch.float64 if args.dtype == "c128" else torch.float32).pin_memory()
    host_state[0] = 1.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(max(1, args.steps // 2)):
        if args.dtype == "c128":
            check(L.qbg_upload(reg._h, host_state.data_ptr(), 1 << n))
        else:  # the device's own element type, no host-side conversion
            check(L.qbg_upload_raw(reg._h, host_state.data_ptr(), S))
        r3 = step()
    torch.cuda.synchronize()
    e2e_state_ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps // 2)
    e2e["with_state_upload"] = {"value": world * 2 * G / (e2e_state_ms / 1e3), "h2d_bytes_per_step": S + 8 * theta.size}

    # ---- per-kernel timing of the dominant kernel (CUDA events around each launch) ----
    peak, peak_src = load_peaks()
    L.qbg_profile_reset()
    L.qbg_profile_enable(1)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    import ctypes
    buf = ctypes.create_string_buffer(1 << 16)
    check(L.qbg_profile_report(buf, len(buf)))
    L.qbg_profile_enable(0)
    kernels = []
    for line in buf.value.decode().strip().splitlines():
        name, cnt, tot, byt, flo = line.split("\t")
        kernels.append({"name": name, "launches": int(cnt), "total_ms": float(tot), "bytes": float(byt),
                        "flops": float(flo)})
    kernels.sort(key=lambda x: -x["total_ms"])
    top = kernels[0] if kernels else None
    roofline = None
    if top:
        per_launch_ms = top["total_ms"] / top["launches"]
        per_launch_bytes = top["bytes"] / top["launches"]
        achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp) and args.dtype == "c128":  # the committed capture is of the c128 metric run
            try:
                traffic = json.load(open(tp)).get(top["name"])
            except Exception:
                traffic = None
        share = top["total_ms"] / sum(k["total_ms"] for k in kernels)
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "kernel": top["name"], "launches_per_step": top["launches"] / 2,
                    "bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms, "share_of_step": share,
                    "peak_source": peak_src,
                    "fp64": fp64_roofline(top, per_launch_ms) if args.dtype == "c128" else None,
                    "per_gate_convention": per_gate_roofline(top, per_launch_ms, G, S, peak),
                    "kernels": [{k2: (round(v, 6) if isinstance(v, float) else v) for k2, v in kk.items()}
                                for kk in kernels[:16]]}
        # whole-step HBM throughput: every kernel's algorithmic bytes of one step over the step time
        step_bytes = sum(k["bytes"] for k in kernels) / 2
        roofline["step"] = {"hbm_gbs": step_bytes / (ms / 1e3) / 1e9, "frac": step_bytes / (ms / 1e3) / 1e9 / peak,
                            "bytes_per_step": step_bytes,
                            "note": "algorithmic bytes of all passes of one step / device step time"}

    # ---- CPU baseline: the reference on this host's cores, bounded sample (rank 0, N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import cpu_baseline as cb
        import oracle as O
        orc, kind = O.reference(), "reference"
        if orc is None:
            orc, kind = O.restatement(), "port"
        k = 2 if args.cpu_budget < 30 else 4
        r = cb.sample_apply_grad(orc, n, d, k, 3, threads=1)
        cpu = {"value": r["value"], "unit": "gates/s", "cores": 1, "kind": kind,
               "sample": r["sample"] + "; 1 core (unbatched state: the reference parallelises over columns only)",
               "cpu_model": cb.cpu_model(), "job_seconds_extrapolated": r["job_seconds_extrapolated"],
               "extrapolation_check": cpu_validation()}

    prog_stats = prog.stats()
    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (zero_state, θ ~ U(0,2π) from Rng(42+rank))",
        "config": workload_config(args),
        "hbm_gbs_algorithmic": hbm_alg, "hbm_frac_algorithmic": hbm_alg / peak,
        "hbm_note": "hbm_*_algorithmic use the per-gate convention (2S per gate per state pass, SURVEY 8(d)): "
                    "> 1 because fusion applies ~34 gates per HBM pass; the real HBM rates are "
                    "roofline.achieved (dominant kernel) and roofline.step (whole step)",
        "energy": float(res.energies[0]),
        "fusion": not args.no_fusion, "prog_stats": prog_stats,
        "e2e": e2e, "gpu_launches": launches, "clocks": ck, "roofline": roofline, "cpu_baseline": cpu,
        "sharded_state": None,
    }

    # The sharded measurement is a secondary key of the metric line: a watchdog on every rank
    # makes sure a stuck exchange (or a peer stuck in NCCL after another rank failed) can never
    # swallow the line or hang the job: rank 0 prints the line once, every rank exits.
    import threading
    printed = threading.Event()

    def emit():
        if rank == 0 and not printed.is_set():
            printed.set()
            print(json.dumps(line), flush=True)

    def _watchdog():
        if line["sharded_state"] is None and not args.no_sharded:
            line["sharded_state"] = {"error": f"timed out after {args.sharded_timeout} s"}
        emit()
        os._exit(0)

    wd = threading.Timer(args.sharded_timeout, _watchdog)
    wd.daemon = True
    wd.start()
    if not args.no_sharded and args.dtype == "c128":
        del reg, prog
        import gc
        gc.collect()
        L.qbg_release_workspace()
        try:
            line["sharded_state"] = sharded_weak_scaling(args, rank, world, pg)
        except Exception as e:  # reported, never fatal to the metric line
            line["sharded_state"] = {"error": f"{type(e).__name__}: {e}"[:300]}

    emit()
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    wd.cancel()


if __name__ == "__main__":
    main()
