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
    is uncomputed back to the input up to rounding) and saves one full-state copy.
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


def faithful_grad(obs: Block, pair) -> np.ndarray:
    """Parameter-shift ("faithful") gradient, exact mode (PAPER eq. shiftrule):
    θ̄_k = ½(⟨O⟩_{θ_k+π/2} − ⟨O⟩_{θ_k−π/2}), summed over the batch.  Every parameter must belong to
    a Rotation with a reflexive generator; Shift / Phase parameters raise UnsupportedError.
    2P device evaluations of the circuit (the forward-mode cost the paper contrasts with AD)."""
    from .blocks import Rotation, dispatch, parameter_nodes, parameters
    from .mmd import MMD, mmd_grad
    if isinstance(obs, MMD):
        return mmd_grad(obs, pair, "shift").param_grads
    reg, circuit = pair
    nodes = parameter_nodes(circuit)
    for nd in nodes:
        if not isinstance(nd, Rotation):
            raise errors.UnsupportedError("faithful_grad: shift rule needs Rotation parameters only")
    theta = parameters(circuit)
    grads = np.empty(theta.size)
    try:
        for k in range(theta.size):
            t = theta.copy()
            t[k] = theta[k] + np.pi / 2
            dispatch(circuit, t)
            ep = float(np.sum(expect(obs, (reg, circuit))))
            t[k] = theta[k] - np.pi / 2
            dispatch(circuit, t)
            em = float(np.sum(expect(obs, (reg, circuit))))
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
