"""Generates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref/libqbref.so, built
from /root/reference/proj/include by oracle/Makefile).  Run here, where the reference exists:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the oracle restatement (and through it the device engine) on boxes where the
reference is absent.  Every case is seeded; re-running reproduces the files bit for bit."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1912_10877_b200 import blocks as B  # noqa: E402
from paper_1912_10877_b200 import circuits as C  # noqa: E402
from paper_1912_10877_b200 import matrix as M  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_gate(rng: np.random.Generator, t: int):
    d = 1 << t
    kind = rng.integers(0, 3)
    if kind == 0:
        return M.Diagonal(np.exp(1j * rng.uniform(0, 2 * np.pi, d)))
    if kind == 1:
        return M.Permutation(rng.permutation(d), np.exp(1j * rng.uniform(0, 2 * np.pi, d)))
    a = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, _ = np.linalg.qr(a)
    return M.Dense(q)


def instruct_cases(ref, count=240, seed=1234, tmin=1, tmax=3, nmax=6):
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(count):
        n = int(rng.integers(max(2, tmin), nmax + 1))
        B_ = int(rng.integers(1, 4))
        t = int(rng.integers(tmin, min(tmax, n) + 1))
        nc = int(rng.integers(0, min(2, n - t) + 1))
        qs = rng.permutation(np.arange(1, n + 1))
        locs, ctrls = [int(v) for v in qs[:t]], [int(v) for v in qs[t:t + nc]]
        cfg = [int(v) for v in rng.integers(0, 2, nc)]
        g = random_gate(rng, t)
        st = rng.normal(size=(B_, 1 << n)) + 1j * rng.normal(size=(B_, 1 << n))
        st /= np.linalg.norm(st, axis=1, keepdims=True)
        out = ref.instruct(st, n, g, locs, ctrls, cfg)
        vals, perm = M.payload(g)
        rows.append(dict(n=n, B=B_, kind=g.kind, dim=g.dim, vals=np.asarray(vals), perm=perm, locs=locs,
                         ctrls=ctrls, cfg=cfg, inp=st, out=out))
    return rows


def lowered(block):
    nodes = B.parameter_nodes(block)
    em = B._Emitter({id(p): k for k, p in enumerate(nodes)})
    B._lower(block, tuple(range(1, block.nqubits + 1)), (), (), em)
    return em


def main():
    ref = O.reference()
    if ref is None:
        raise SystemExit("oracle/_ref/libqbref.so missing: build it with `make -C oracle` where /root/reference exists")
    # 1. instruct (register.hpp:392-408)
    rows = instruct_cases(ref)
    obj = np.empty(len(rows), dtype=object)
    for k, r in enumerate(rows):
        obj[k] = r
    np.save(os.path.join(OUT, "instruct_cases.npy"), obj, allow_pickle=True)
    # 4- and 5-qubit gates (the dense fallback's widest blocks, register.hpp:371-384)
    rows = instruct_cases(ref, count=80, seed=4545, tmin=4, tmax=5, nmax=8)
    obj = np.empty(len(rows), dtype=object)
    for k, r in enumerate(rows):
        obj[k] = r
    np.save(os.path.join(OUT, "instruct_cases_t45.npy"), obj, allow_pickle=True)

    # 2. Rng / dispatch("random") / rand_state
    r = ref.rng(42)
    uni = np.array([r.uniform() for _ in range(64)])
    bits = np.array([r.bits() for _ in range(16)], dtype=np.uint64)
    gau = np.array([r.gauss() for _ in range(32)])
    theta = ref.dispatch_random(75, 42)
    rs = ref.rand_state(5, 3, 42)
    np.savez(os.path.join(OUT, "rng.npz"), uniform=uni, bits=bits, gauss=gau, dispatch_random=theta,
             rand_state_5_3_42=rs)

    # 3. expect / expect_grad: variational_circuit(4,3) + heisenberg(4), App G (periodic heisenberg(3))
    circ = C.variational_circuit(4, 3)
    th = ref.dispatch_random(B.nparameters(circ), 42)
    B.dispatch(circ, th)
    h = C.heisenberg(4)
    em = lowered(circ)
    st0 = ref.rand_state(4, 2, 5)
    e, g, psi, sg = ref.expect_grad(st0, 4, em, th, B.pauli_terms(h))
    fwd = ref.apply_program(st0, 4, em, th)
    appg = B.chain(B.put(3, 2, B.Rx(0.5)), B.control(3, 2, 1, B.Ry(0.7)), B.put(3, (1, 2), B.rot(B.kron(B.X, B.X), 0.8)))
    eg, gg, _, _ = ref.expect_grad(O.Oracle.zero_state(3), 3, lowered(appg), B.parameters(appg),
                                   B.pauli_terms(C.heisenberg(3, periodic=True)))
    np.savez(os.path.join(OUT, "ad.npz"), theta=th, state_in=st0, forward=fwd, energies=e, grads=g, psi_back=psi,
             state_grad=sg, appg_energy=eg, appg_grads=gg)

    # 4. measurement (register.hpp:414-493)
    st = ref.rand_state(6, 2, 9)
    st = ref.instruct(st, 6, M.h(), [2])
    r = ref.rng(11)
    samples = ref.measure(st, 6, 6, 50, r)
    r2 = ref.rng(12)
    hits, collapsed = ref.measure_collapse(st, 6, 6, r2)
    probs = ref.probabilities(st, 6, 6, 1)
    np.savez(os.path.join(OUT, "measure.npz"), state=st, samples=samples, hits=hits, collapsed=collapsed, probs1=probs)

    # 5. focus / relax (register.hpp:156-177)
    st = ref.rand_state(6, 2, 21)
    foc = ref.focus(st, 6, [3, 6, 1, 2])
    np.savez(os.path.join(OUT, "focus.npz"), state=st, locs=np.array([3, 6, 1, 2]), focused=foc)
    # 6. QBREG1 state file written by the reference (register.hpp:181-188), nactive = 3 of 4
    st = ref.rand_state(4, 2, 33)
    ref.save(st, 4, 3, os.path.join(OUT, "state_qbreg1.bin"))
    np.save(os.path.join(OUT, "state_qbreg1_amps.npy"), st)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
