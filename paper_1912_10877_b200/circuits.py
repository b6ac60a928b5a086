"""The two circuit-zoo members on the hot path: the hardware-efficient
variational circuit and the Heisenberg chain.  They ARE the BASELINE workloads."""
from __future__ import annotations

import math

from .blocks import H, Rx, Rz, X, Y, Z, Add, Block, chain, control, put, shift


def variational_circuit(n: int, depth: int) -> Block:
    """an initial Rx layer, then ``depth`` layers of a CNOT ring
    (control i -> target i mod n + 1, i = 1..n) followed by Rz, Rx, Rz on every qubit.
    Gate count Rz 2nd, Rx nd + n, CNOT nd; nparameters 3nd + n."""
    if n < 2 or depth < 1:
        raise ValueError("variational_circuit: need n >= 2 and depth >= 1")
    blocks = [put(n, q, Rx(0.0)) for q in range(1, n + 1)]
    for _ in range(depth):
        for i in range(1, n + 1):
            blocks.append(control(n, i, i % n + 1, X))
        for q in range(1, n + 1):
            blocks.append(put(n, q, chain(Rz(0.0), Rx(0.0), Rz(0.0))))
    return chain(n, *blocks)


def heisenberg(n: int, periodic: bool = False) -> Block:
    """Listing 6 / SPEC.md:557-561: Σ_bonds (XX + YY + ZZ).  Open chain by default (SPEC);
    ``periodic=True`` adds the (n, 1) bond (YaoExtensions' default, used by App G)."""
    if n < 2:
        raise ValueError("heisenberg: need n >= 2")
    bonds = [(i, i + 1) for i in range(1, n)]
    if periodic:
        bonds.append((n, 1))
    terms = []
    for i, j in bonds:
        for s in (X, Y, Z):
            terms.append(put(n, i, s) * put(n, j, s))
    return Add(terms)


def qft(n: int) -> Block:
    """Listing 1: chain of hcphases(n, i) = chain(H on i, cphase(j, i) for j = i+1..n) with
    cphase(j, i) = control(j, i => shift(2π / 2^(j-i+1)))."""
    outer = []
    for i in range(1, n + 1):
        inner = [put(n, i, H)]
        for j in range(i + 1, n + 1):
            inner.append(control(n, j, i, shift(2 * math.pi / (1 << (j - i + 1)))))
        outer.append(chain(n, *inner))
    return chain(n, *outer)
