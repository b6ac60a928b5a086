"""Bounded CPU timing of the apply+grad workload on the oracle — TEST INFRASTRUCTURE ONLY
(bench.py's cpu_baseline and --impl reference legs).

The full 25-qubit job takes ~10 minutes on one core, so it is timed on a bounded sample of
the same workload and extrapolated per unit of work:
  * forward  : k CNOTs of the ring + the k following Rz·Rx·Rz rotation triples of layer 1
               (the layer's own 1:3 CNOT:rotation mix), applied to the 25-qubit state;
  * backward : the reverse loop (uncompute ψ, back-propagate φ̄, mat_back gradient) over
               the same 4k instructions;
  * seed     : m Pauli terms of heisenberg(n) applied to ψ (φ̄ = Oψ) plus the energy.
  T_job ≈ G/(4k)·(t_fwd + t_bwd) + T/m·t_seed;  value = 2G / T_job  (gates/s, fwd + bwd).
"""
from __future__ import annotations

import os
import time

import numpy as np


def _lowered(block, ops_idx=None):
    from paper_1912_10877_b200 import blocks as B
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    if ops_idx is not None:
        em.ops = [em.ops[i] for i in ops_idx]
    return em


def sample_apply_grad(orc, n: int, depth: int, k: int, m: int, threads: int = 1, seed: int = 42) -> dict:
    from paper_1912_10877_b200 import blocks as B
    from paper_1912_10877_b200 import circuits as C
    circ = C.variational_circuit(n, depth)
    th = orc.dispatch_random(B.nparameters(circ), seed)
    full = _lowered(circ)
    G = len(full.ops)
    terms = B.pauli_terms(C.heisenberg(n))
    T = len(terms)
    k = max(1, min(k, n))
    m = max(1, min(m, T))
    idx = list(range(n, n + k)) + list(range(2 * n, 2 * n + 3 * k))
    em = _lowered(circ, idx)
    orc.set_threads(threads)
    psi = orc.zero_state(n)
    # compute-only timers inside the library (steady_clock around the instruct loops), so the
    # ctypes/Register marshalling of the 2^n buffers is not charged to the reference
    psi = orc.apply_program(psi, n, em, th)
    t_fwd = orc.last_kernel_seconds()
    phi, _ = orc.obs_apply(psi, terms[:m])
    t_seed = orc.last_kernel_seconds()
    grads = np.zeros(max(1, len(th)))
    orc.backward(psi, phi, n, em, th, grads)
    t_bwd = orc.last_kernel_seconds()
    t_job = G / (4 * k) * (t_fwd + t_bwd) + T / m * t_seed
    return {
        "value": 2 * G / t_job,
        "unit": "gates/s",
        "job_seconds_extrapolated": t_job,
        "sample_seconds": t_fwd + t_bwd + t_seed,
        "sample": (f"variational_circuit({n},{depth}) apply+grad, heisenberg({n}) open: timed {4 * k} "
                   f"layer-1 instructions ({k} CNOT + {3 * k} rotations) forward and backward and "
                   f"{m}/{T} seed terms on the {n}-qubit state; extrapolated per instruction / term to "
                   f"G={G}, T={T}"),
        "t_fwd": t_fwd, "t_bwd": t_bwd, "t_seed": t_seed, "k": k, "m": m,
    }


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def nproc() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
