"""Maximum mean discrepancy loss of a circuit's output distribution (SPEC.md:446-449 MMDLoss,
497-505 mmd_expect / mmd_grad; §3.2 and Listing 12).

    kf  = brbf_kernel(2.0)
    mmd = MMD(kf, target_p)
    g   = expect_grad(mmd, (zero_state(n), circuit))     # reverse mode through p = |ψ|²
    g2  = mmd_grad(mmd, (zero_state(n), circuit), mode="shift")

L = Σ_{x,y} K(x,y)(p−q)_x(p−q)_y with K(x,y) = Σ_σ exp(−(x−y)²/(2σ²)) over the integer
distance |x−y|.  Every evaluation runs on the device (``qbg_mmd_*`` in include/qbg.h): the
Toeplitz kernel is applied as an exact banded convolution, the reverse seed is
φ̄ = 2 (K(p−q)) ⊙ ψ, and the shift rule uses the cross statistic
E_{x∼p±, y∼p} K − E_{x∼p±, y∼q} K of the paper's estimator."""
from __future__ import annotations

import ctypes

import numpy as np

from . import errors
from ._capi import check, lib
from .ad import GradResult
from .blocks import Block, Rotation, apply, compile_block, dispatch, parameter_nodes, parameters
from .register import Register


class RBFKernel:
    """Radial-basis mixture over the integer distance: K(x,y) = Σ_σ exp(−(x−y)²/(2σ²))."""

    def __init__(self, sigmas):
        self.sigmas = np.atleast_1d(np.asarray(sigmas, dtype=np.float64)).copy()
        if self.sigmas.size == 0 or np.any(~(self.sigmas > 0)):
            raise errors.ValidationError("brbf_kernel: bandwidths must be > 0")

    def __call__(self, x, y):
        d2 = (np.asarray(x, dtype=np.float64) - np.asarray(y, dtype=np.float64)) ** 2
        return sum(np.exp(-d2 / (2.0 * s * s)) for s in self.sigmas)


def brbf_kernel(*sigmas) -> RBFKernel:
    """Yao's ``brbf_kernel(σ)`` (Listing 12): the RBF mixture over basis-index distance."""
    return RBFKernel(sigmas)


class MMD:
    """MMDLoss(kernel, target_p).  target_p: 2^n probabilities summing to 1."""

    def __init__(self, kernel: RBFKernel, target_p):
        q = np.ascontiguousarray(target_p, dtype=np.float64)
        n = int(q.size).bit_length() - 1
        if q.ndim != 1 or q.size != (1 << n):
            raise errors.ShapeError("MMD: target_p must have length 2^n")
        self.kernel, self.target_p, self.nqubits = kernel, q, n
        s = np.ascontiguousarray(kernel.sigmas)
        h = ctypes.c_void_p()
        check(lib().qbg_mmd_create(n, q.ctypes.data, s.ctypes.data, s.size, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().qbg_mmd_destroy(h)
            except Exception:
                pass

    @property
    def band(self) -> int:
        b = ctypes.c_int32()
        check(lib().qbg_mmd_band(self._h, ctypes.byref(b)))
        return b.value


def _out(reg):
    return np.empty(reg.nbatch)


def mmd_expect(loss: MMD, reg_or_pair) -> np.ndarray:
    """Per-batch squared MMD of p = |ψ|² against target_p (mmd_expect)."""
    if isinstance(reg_or_pair, tuple):
        reg, circuit = reg_or_pair
        reg = reg.copy()
        apply(reg, circuit)
    else:
        reg = reg_or_pair
    out = _out(reg)
    check(lib().qbg_mmd_loss(reg._h, loss._h, out.ctypes.data))
    return out


def mmd_seed(loss: MMD, psi: Register, adj: Register | None = None):
    """(loss per batch, φ̄ = ∂L/∂ψ* = 2 (K(p−q)) ⊙ ψ)."""
    if adj is None:
        adj = Register(psi.nqubits, psi.nbatch, dtype=psi.dtype)
    out = _out(psi)
    check(lib().qbg_mmd_seed(psi._h, loss._h, adj._h, out.ctypes.data))
    return out, adj


def mmd_cross(loss: MMD, a: Register, reg: Register) -> np.ndarray:
    """Σ_{x,y} K(x,y) p^a(x) (p(y) − q(y)) per batch (the shift-rule statistic)."""
    out = _out(reg)
    check(lib().qbg_mmd_cross(a._h, reg._h, loss._h, out.ctypes.data))
    return out


def mmd_grad(loss: MMD, pair, mode: str = "reverse", want_state_grad: bool = False, inplace: bool = False):
    """mmd_grad(loss, reg => circuit, mode).

    reverse: forward once, seed φ̄ = 2K(p−q)⊙ψ, reverse pass (returns GradResult).
    shift  : paper §3.2, per rotation parameter θ_k
             ∂L/∂θ_k = Σ_b [E_{x∼p_{θ+π/2}, y∼p} K − E_{x∼p_{θ+π/2}, y∼q} K] − [same at θ−π/2]
             (returns GradResult without state_grad); 2P + 1 device circuit evaluations."""
    reg, circuit = pair
    if circuit.nqubits != reg.nactive or loss.nqubits != reg.nactive:
        raise errors.ShapeError("mmd_grad: circuit output dimension differs from target_p")
    if mode == "reverse":
        p = compile_block(circuit)
        vals = _out(reg)
        grads = np.zeros(max(1, p.nparams))
        sg = Register(reg.nqubits, reg.nbatch, dtype=reg.dtype) if want_state_grad else None
        check(lib().qbg_mmd_grad(reg._h, p._h, loss._h, 1 if inplace else 0, vals.ctypes.data, grads.ctypes.data,
                                 sg._h if sg is not None else None))
        return GradResult(vals, grads[: p.nparams], sg)
    if mode != "shift":
        raise errors.ValidationError(f"mmd_grad: unknown mode {mode!r} (reverse | shift)")
    for nd in parameter_nodes(circuit):
        if not isinstance(nd, Rotation):
            raise errors.UnsupportedError("mmd_grad(shift): the shift rule needs Rotation parameters only")
    theta = parameters(circuit)
    psi = reg.copy()
    apply(psi, circuit)
    vals = mmd_expect(loss, psi)
    grads = np.empty(theta.size)
    tmp = Register(reg.nqubits, reg.nbatch, dtype=reg.dtype)
    try:
        for k in range(theta.size):
            acc = 0.0
            for sgn in (1.0, -1.0):
                t = theta.copy()
                t[k] = theta[k] + sgn * np.pi / 2
                dispatch(circuit, t)
                tmp.assign(reg)
                apply(tmp, circuit)
                acc += sgn * float(np.sum(mmd_cross(loss, tmp, psi)))
            grads[k] = acc
    finally:
        dispatch(circuit, theta)
    return GradResult(vals, grads)
