"""Expectation values and reversible-AD gradients (Yao.AD) on the device.

``expect_grad(obs, (reg, circuit))`` runs forward once, seeds φ̄ = O|ψ⟩ and walks the
circuit backwards uncomputing ψ and back-propagating φ̄, with at most
two extra full states live regardless of depth."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import errors
from ._capi import check, lib
from .blocks import Block, apply, compile_block, compile_observable
from .register import Register


@dataclass
class GradResult:
    energies: np.ndarray     # per batch <O>
    param_grads: np.ndarray  # summed over the batch, parameters() order
    state_grad: Register | None = None  # adjoint of the input state


def _pair(reg_or_pair):
    if isinstance(reg_or_pair, tuple):
        return reg_or_pair
    return reg_or_pair, None


def expect(obs: Block, reg_or_pair) -> np.ndarray:
    """expect(O, reg) or expect(O, (reg, circuit)) -> per-batch real <O>.
    An :class:`~paper_1912_10877_b200.mmd.MMD` loss in place of O gives the per-batch MMD."""
    from .mmd import MMD, mmd_expect
    if isinstance(obs, MMD):
        return mmd_expect(obs, reg_or_pair)
    reg, circuit = _pair(reg_or_pair)
    if circuit is not None:
        reg = reg.copy()
        apply(reg, circuit)
    o = compile_observable(obs)
    out = np.empty(reg.nbatch)
    check(lib().qbg_expect(reg._h, o._h, out.ctypes.data))
    return out


def obs_apply(obs: Block, reg: Register, out: Register | None = None) -> Register:
    """|out> = O |reg> for a Pauli-sum observable."""
    o = compile_observable(obs)
    if out is None:
        out = Register(reg.nqubits, reg.nbatch, dtype=reg.dtype)
    check(lib().qbg_obs_apply(reg._h, o._h, out._h))
    return out


def expect_grad(obs: Block, pair, want_state_grad: bool = False, inplace: bool = False) -> GradResult:
    """expect'(O, reg => circuit).  ``inplace`` runs on ``reg`` itself (it
    is uncomputed back to the input up to rounding) and saves one full-state copy.  With the
    checkpointed design (default when its checkpoints fit, see set_checkpointing) the register is
    never modified, in place or not.
    ``obs`` may be an MMD loss (Listing 12: expect'(mmd, zero_state(n)=>circuit))."""
    from .mmd import MMD, mmd_grad
    if isinstance(obs, MMD):
        return mmd_grad(obs, pair, "reverse", want_state_grad, inplace)
    from .blocks import has_time_evolution
    if has_time_evolution(pair[1]):
        return _expect_grad_segmented(obs, pair, want_state_grad)
    reg, circuit = pair
    if circuit.nqubits != reg.nactive or obs.nqubits != reg.nactive:
        raise errors.ShapeError("expect': block qubit count differs from active qubits")
    p = compile_block(circuit)
    o = compile_observable(obs)
    energies = np.empty(reg.nbatch)
    grads = np.zeros(max(1, p.nparams))
    sg = Register(reg.nqubits, reg.nbatch, dtype=reg.dtype) if want_state_grad else None
    check(lib().qbg_expect_grad(reg._h, p._h, o._h, 1 if inplace else 0, energies.ctypes.data, grads.ctypes.data,
                                sg._h if sg is not None else None))
    return GradResult(energies, grads[: p.nparams], sg)


def _controlled_param(b, under=False) -> bool:
    """A rotation under a Control node has the generator P_ctrl ⊗ Σ, which is not reflexive."""
    from .blocks import Control, Phase, Rotation, Shift
    if isinstance(b, (Rotation, Shift, Phase)):
        return under
    return any(_controlled_param(c, under or isinstance(b, Control)) for c in b.subblocks())


def eigenbasis(obs: Block):
    """eigenbasis(O) -> (E, U) with O = U E U† (SPEC.md blocks.eigenbasis, Listing 10) for a Pauli
    string or a sum of them: per qubit X -> (Z, H), Y -> (Z, chain(H, S)), Z -> (Z, I).  Returns a
    list of (E_terms, U) measurement settings: the terms are grouped qubit-wise compatibly (all
    terms of a group share the basis of every qubit they touch), E_terms are the (c, zmask)
    diagonal terms in that basis, and U is the basis-change circuit (apply U† = dagger(U) before
    sampling in the computational basis)."""
    from .blocks import H as Hg, S as Sg, chain, dagger, pauli_terms, put
    n = obs.nqubits
    groups = []  # [(basis dict qubit -> 'X'|'Y'|'Z', [(c, support mask)])]
    for c, x, z in pauli_terms(obs):
        basis = {}
        for q in range(n):
            if (x >> q) & 1:
                basis[q] = "Y" if (z >> q) & 1 else "X"
            elif (z >> q) & 1:
                basis[q] = "Z"
        for gb, ts in groups:
            if all(gb.get(q, b) == b for q, b in basis.items()):
                gb.update(basis)
                ts.append((c, x | z))
                break
        else:
            groups.append((dict(basis), [(c, x | z)]))
    out = []
    for gb, ts in groups:
        blocks = []
        for q, b in sorted(gb.items()):
            if b == "X":
                blocks.append(put(n, q + 1, Hg))
            elif b == "Y":
                blocks.append(put(n, q + 1, chain(Hg, Sg)))
        U = chain(n, *blocks) if blocks else None
        out.append((ts, U, None if U is None else dagger(U)))
    return out


def sampled_expect(obs: Block, reg: Register, nshots: int, rng=None) -> np.ndarray:
    """⟨O⟩ per batch estimated from nshots computational-basis samples per measurement setting
    (Listing 10 pipeline): rotate a copy by U† of each eigenbasis group, sample
    on the device (bit-exact stream, register.hpp:436-459), average the diagonal eigenvalues
    Σ c (-1)^{popcount(bits & support)}."""
    from .register import measure
    est = np.zeros(reg.nbatch)
    for ts, _, Udag in eigenbasis(obs):
        work = reg.copy()
        if Udag is not None:
            apply(work, Udag)
        bits = measure(work, nshots, rng)  # (nbatch, nshots)
        for c, m in ts:
            par = np.zeros(bits.shape, dtype=np.int64)
            v = bits & np.uint64(m)
            while v.any():  # popcount parity
                par ^= (v & np.uint64(1)).astype(np.int64)
                v = v >> np.uint64(1)
            est += np.real(c) * (1.0 - 2.0 * par).mean(axis=1)
    return est


def faithful_grad(obs: Block, pair, nshots: int | None = None, rng=None) -> np.ndarray:
    """Parameter-shift ("faithful") gradient (PAPER eq. shiftrule):
    θ̄_k = ½(⟨O⟩_{θ_k+π/2} − ⟨O⟩_{θ_k−π/2}), summed over the batch.  Every parameter must belong to
    a Rotation with a reflexive generator; Shift / Phase parameters raise UnsupportedError.
    2P device evaluations of the circuit (the forward-mode cost the paper contrasts with AD).
    ``nshots=None`` is the exact mode (expect); an integer estimates each ⟨O⟩ from nshots samples
    per eigenbasis setting (``sampled_expect``; ``rng`` a :class:`Rng`, default Rng(42))."""
    from .blocks import Rotation, dispatch, parameter_nodes, parameters
    from .mmd import MMD, mmd_grad
    if isinstance(obs, MMD):
        return mmd_grad(obs, pair, "shift").param_grads
    reg, circuit = pair
    nodes = parameter_nodes(circuit)
    for nd in nodes:
        if not isinstance(nd, Rotation):
            raise errors.UnsupportedError("faithful_grad: shift rule needs Rotation parameters only")
    if _controlled_param(circuit):
        raise errors.UnsupportedError("faithful_grad: a controlled rotation's generator is not reflexive (no shift rule)")
    theta = parameters(circuit)
    grads = np.empty(theta.size)
    if nshots is not None:
        from .register import Rng
        rng = rng if rng is not None else Rng(42)

    def value():
        if nshots is None:
            return float(np.sum(expect(obs, (reg, circuit))))
        psi = reg.copy()
        apply(psi, circuit)
        return float(np.sum(sampled_expect(obs, psi, nshots, rng)))

    try:
        for k in range(theta.size):
            t = theta.copy()
            t[k] = theta[k] + np.pi / 2
            dispatch(circuit, t)
            ep = value()
            t[k] = theta[k] - np.pi / 2
            dispatch(circuit, t)
            em = value()
            grads[k] = 0.5 * (ep - em)
    finally:
        dispatch(circuit, theta)
    return grads


def backward(psi: Register, adj: Register, circuit: Block, grads: np.ndarray | None = None) -> np.ndarray:
    """apply_back through a whole circuit: uncomputes psi, back-propagates
    adj, and adds the parameter gradient into ``grads``."""
    p = compile_block(circuit)
    g = np.zeros(max(1, p.nparams)) if grads is None else np.ascontiguousarray(grads, dtype=np.float64)
    check(lib().qbg_backward(psi._h, adj._h, p._h, g.ctypes.data))
    return g[: p.nparams]


def _expect_grad_segmented(obs: Block, pair, want_state_grad: bool) -> GradResult:
    """expect' through circuits with time_evolve nodes (SPEC.md:479-487 + the TimeEvolution design
    decision): the gate segments run the device reverse pass (qbg_backward); a TimeEvolution
    e^{-iHt} contributes t̄ = 2 Im<φ̄|H|ψ> (taken after it, summed over the batch) and is then
    uncomputed on ψ and φ̄ by e^{+iHt} (two more Krylov applications)."""
    from .blocks import apply_hamiltonian, evolve, parameter_nodes, segments
    reg, circuit = pair
    if circuit.nqubits != reg.nactive or obs.nqubits != reg.nactive:
        raise errors.ShapeError("expect': block qubit count differs from active qubits")
    index = {id(nd): k for k, nd in enumerate(parameter_nodes(circuit))}
    grads = np.zeros(len(index))
    psi = reg.copy()
    segs = segments(circuit)
    for kind, seg in segs:
        if kind == "te":
            evolve(psi, seg.hamiltonian, seg.theta)
        else:
            check(lib().qbg_apply(psi._h, compile_block(seg)._h))
    adj = obs_apply(obs, psi)
    energies = np.real(psi.inner(adj))
    tmp = None
    for kind, seg in reversed(segs):
        if kind == "te":
            tmp = apply_hamiltonian(seg.hamiltonian, psi, tmp)
            grads[index[id(seg)]] += 2.0 * float(np.sum(np.imag(adj.inner(tmp))))
            evolve(psi, seg.hamiltonian, -seg.theta)
            evolve(adj, seg.hamiltonian, -seg.theta)
        else:
            g = backward(psi, adj, seg)
            for k, nd in enumerate(parameter_nodes(seg)):
                grads[index[id(nd)]] += g[k]
    return GradResult(energies, grads, adj if want_state_grad else None)
