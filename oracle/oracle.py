"""ctypes wrapper of the CPU oracles — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module, and only as the checker (never as the thing measured or shipped).

Two libraries with the same C ABI (orc_*):
  * ``restatement()`` -> oracle/libqbg_oracle.so, the plain C++ restatement (qbg_oracle.cpp);
  * ``reference()``   -> oracle/_ref/libqbref.so, the same entry points running the
    UNMODIFIED reference headers (ref_driver.cpp); None where it was never built.
States use the reference layout: complex128 arrays of shape (B, 2**n), batch slowest.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT = os.path.join(HERE, "libqbg_oracle.so")
REFERENCE = os.path.join(HERE, "_ref", "libqbref.so")


class Oracle:
    def __init__(self, path: str):
        self.path = path
        L = ctypes.CDLL(path)
        P = c_void_p
        sig = {
            "orc_last_error": (c_char_p, []),
            "orc_rng_new": (P, [c_uint64]), "orc_rng_free": (None, [P]),
            "orc_rng_split_label": (P, [P, c_char_p]), "orc_rng_uniform": (c_double, [P]),
            "orc_rng_uniform_range": (c_double, [P, c_double, c_double]), "orc_rng_gauss": (c_double, [P]),
            "orc_rng_bits": (c_uint64, [P]), "orc_dispatch_random": (None, [P, c_int64, c_uint64]),
            "orc_rand_state": (c_int, [P, c_int, c_int64, c_uint64]),
            "orc_instruct": (c_int, [P, c_int, c_int, c_int64, c_int, c_int, P, P, P, c_int, P, P, c_int]),
            "orc_apply_program": (c_int, [P, c_int, c_int64, P, c_int64, P, P, P, c_int]),
            "orc_inner": (c_int, [P, P, c_int, c_int64, P]), "orc_norm": (c_int, [P, c_int, c_int64, P]),
            "orc_obs_apply": (c_int, [P, c_int, c_int64, P, c_int64, P, P]),
            "orc_expect": (c_int, [P, c_int, c_int64, P, c_int64, P]),
            "orc_expect_grad": (c_int, [P, c_int, c_int64, P, c_int64, P, P, P, c_int64, P, c_int64, P, P, P, P]),
            "orc_probabilities": (c_int, [P, c_int, c_int, c_int64, P]),
            "orc_measure": (c_int, [P, c_int, c_int, c_int64, c_int64, P, P]),
            "orc_measure_collapse": (c_int, [P, c_int, c_int, c_int64, P, P]),
            "orc_focus": (c_int, [P, c_int, c_int64, P, c_int]), "orc_relax": (c_int, [P, c_int, c_int64, P, c_int]),
            "orc_backward": (c_int, [P, P, c_int, c_int64, P, c_int64, P, P, P, P]),
            "orc_set_threads": (None, [c_int]), "orc_last_kernel_seconds": (c_double, []),
            "orc_save": (c_int, [P, c_int, c_int, c_int64, c_char_p]),
            "orc_load": (c_int, [c_char_p, P, c_int64, POINTER(c_int), POINTER(c_int), POINTER(c_int64)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        self.L = L

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.orc_last_error().decode())

    # ---- rng ----
    def rng(self, seed=42):
        return _Rng(self, self.L.orc_rng_new(seed))

    def dispatch_random(self, nparams: int, seed: int = 42) -> np.ndarray:
        th = np.empty(nparams)
        self.L.orc_dispatch_random(th.ctypes.data, nparams, seed)
        return th

    # ---- states ----
    def rand_state(self, n, B=1, seed=42):
        st = np.empty((B, 1 << n), dtype=np.complex128)
        self._chk(self.L.orc_rand_state(st.ctypes.data, n, B, seed))
        return st

    @staticmethod
    def zero_state(n, B=1):
        st = np.zeros((B, 1 << n), dtype=np.complex128)
        st[:, 0] = 1
        return st

    def instruct(self, st, n, mat, locs, ctrls=(), cfg=(), nactive=None):
        """mat: paper_1912_10877_b200.matrix.Matrix (payload via matrix.payload)."""
        from paper_1912_10877_b200.matrix import payload
        st = np.ascontiguousarray(st, dtype=np.complex128).copy()
        B = st.shape[0]
        vals, perm = payload(mat)
        vals = np.ascontiguousarray(vals, dtype=np.complex128)
        perm = np.ascontiguousarray(perm if perm is not None else np.zeros(1, np.int64), dtype=np.int64)
        la = np.array(list(locs) or [0], dtype=np.int32)
        ca = np.array(list(ctrls) or [0], dtype=np.int32)
        fa = np.array(list(cfg) or [0], dtype=np.int32)
        self._chk(self.L.orc_instruct(st.ctypes.data, n, n if nactive is None else nactive, B, mat.kind, mat.dim,
                                      vals.ctypes.data, perm.ctypes.data, la.ctypes.data, len(locs), ca.ctypes.data,
                                      fa.ctypes.data, len(ctrls)))
        return st

    def apply_program(self, st, n, em, theta, adjoint=False):
        """em: blocks._Emitter (ops/vals/perms of a lowered block)."""
        st = np.ascontiguousarray(st, dtype=np.complex128).copy()
        ops, vals, perms = _pack(em)
        th = np.ascontiguousarray(theta if len(theta) else [0.0], dtype=np.float64)
        self._chk(self.L.orc_apply_program(st.ctypes.data, n, st.shape[0], ops, len(em.ops), vals.ctypes.data,
                                           perms.ctypes.data, th.ctypes.data, 1 if adjoint else 0))
        return st

    def inner(self, a, b):
        out = np.empty(2 * a.shape[0])
        n = int(np.log2(a.shape[1]))
        self._chk(self.L.orc_inner(np.ascontiguousarray(a).ctypes.data, np.ascontiguousarray(b).ctypes.data, n,
                                   a.shape[0], out.ctypes.data))
        return out[0::2] + 1j * out[1::2]

    def obs_apply(self, st, terms):
        st = np.ascontiguousarray(st, dtype=np.complex128)
        n = int(np.log2(st.shape[1]))
        arr = _terms(terms)
        phi = np.empty_like(st)
        e = np.empty(st.shape[0])
        self._chk(self.L.orc_obs_apply(st.ctypes.data, n, st.shape[0], arr, len(terms), phi.ctypes.data,
                                       e.ctypes.data))
        return phi, e

    def expect_grad(self, st, n, em, theta, terms):
        st = np.ascontiguousarray(st, dtype=np.complex128)
        B = st.shape[0]
        ops, vals, perms = _pack(em)
        th = np.ascontiguousarray(theta if len(theta) else [0.0], dtype=np.float64)
        e = np.empty(B)
        g = np.zeros(max(1, len(theta)))
        psi = np.empty_like(st)
        sg = np.empty_like(st)
        self._chk(self.L.orc_expect_grad(st.ctypes.data, n, B, ops, len(em.ops), vals.ctypes.data, perms.ctypes.data,
                                         th.ctypes.data, len(theta), _terms(terms), len(terms), e.ctypes.data,
                                         g.ctypes.data, psi.ctypes.data, sg.ctypes.data))
        return e, g[: len(theta)], psi, sg

    def backward(self, psi, phi, n, em, theta, grads):
        """In place on psi/phi (complex128 (B, 2**n) C-contiguous arrays)."""
        ops, vals, perms = _pack(em)
        th = np.ascontiguousarray(theta if len(theta) else [0.0], dtype=np.float64)
        self._chk(self.L.orc_backward(psi.ctypes.data, phi.ctypes.data, n, psi.shape[0], ops, len(em.ops),
                                      vals.ctypes.data, perms.ctypes.data, th.ctypes.data, grads.ctypes.data))

    def save(self, st, n, nactive, path):
        st = np.ascontiguousarray(st, dtype=np.complex128)
        self._chk(self.L.orc_save(st.ctypes.data, n, nactive, st.shape[0], str(path).encode()))

    def load(self, path, cap=1 << 22):
        buf = np.empty(cap, dtype=np.complex128)
        n, na, B = c_int(), c_int(), c_int64()
        self._chk(self.L.orc_load(str(path).encode(), buf.ctypes.data, cap, ctypes.byref(n), ctypes.byref(na),
                                  ctypes.byref(B)))
        return buf[: (1 << n.value) * B.value].reshape(B.value, 1 << n.value).copy(), n.value, na.value

    def last_kernel_seconds(self) -> float:
        """Compute time of the last apply_program / obs_apply / backward call, excluding the
        host marshalling of the reference Register."""
        return self.L.orc_last_kernel_seconds()

    def set_threads(self, k):
        self.L.orc_set_threads(k)

    def probabilities(self, st, n, nactive, b=0):
        p = np.empty(1 << nactive)
        self._chk(self.L.orc_probabilities(np.ascontiguousarray(st).ctypes.data, n, nactive, b, p.ctypes.data))
        return p

    def measure(self, st, n, nactive, nshots, rng):
        B = st.shape[0]
        out = np.empty(B * nshots, dtype=np.uint64)
        self._chk(self.L.orc_measure(np.ascontiguousarray(st).ctypes.data, n, nactive, B, nshots, rng.h,
                                     out.ctypes.data))
        return out.reshape(B, nshots)

    def measure_collapse(self, st, n, nactive, rng):
        st = np.ascontiguousarray(st, dtype=np.complex128).copy()
        out = np.empty(st.shape[0], dtype=np.uint64)
        self._chk(self.L.orc_measure_collapse(st.ctypes.data, n, nactive, st.shape[0], rng.h, out.ctypes.data))
        return out, st

    def focus(self, st, n, locs):
        st = np.ascontiguousarray(st, dtype=np.complex128).copy()
        la = np.array(locs, dtype=np.int32)
        self._chk(self.L.orc_focus(st.ctypes.data, n, st.shape[0], la.ctypes.data, len(locs)))
        return st

    def relax(self, st, n, locs):
        st = np.ascontiguousarray(st, dtype=np.complex128).copy()
        la = np.array(locs, dtype=np.int32)
        self._chk(self.L.orc_relax(st.ctypes.data, n, st.shape[0], la.ctypes.data, len(locs)))
        return st


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Rng:
    def __init__(self, o, h):
        self.o, self.h = o, h

    def __del__(self):
        if self.h:
            self.o.L.orc_rng_free(self.h)
            self.h = None

    def uniform(self, lo=None, hi=None):
        return self.o.L.orc_rng_uniform(self.h) if lo is None else self.o.L.orc_rng_uniform_range(self.h, lo, hi)

    def gauss(self):
        return self.o.L.orc_rng_gauss(self.h)

    def bits(self):
        return self.o.L.orc_rng_bits(self.h)

    def split(self, label):
        return _Rng(self.o, self.o.L.orc_rng_split_label(self.h, label.encode()))


def _pack(em):
    from paper_1912_10877_b200._capi import QbgOp
    ops = (QbgOp * max(1, len(em.ops)))(*em.ops)
    vals = np.ascontiguousarray(np.array(em.vals or [0j], dtype=np.complex128))
    perms = np.ascontiguousarray(np.array(em.perms or [0], dtype=np.int64))
    return ops, vals, perms


def _terms(terms):
    from paper_1912_10877_b200._capi import QbgPauliTerm
    arr = (QbgPauliTerm * max(1, len(terms)))()
    for k, (c, x, z) in enumerate(terms):
        arr[k] = QbgPauliTerm(complex(c).real, complex(c).imag, x, z)
    return arr


_cache = {}


def restatement() -> Oracle:
    if "r" not in _cache:
        _cache["r"] = Oracle(RESTATEMENT)
    return _cache["r"]


def reference() -> Oracle | None:
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REFERENCE) if os.path.exists(REFERENCE) else None
    return _cache["ref"]


# ---- MMD loss (SPEC.md:446-449 MMDLoss; 497-505 mmd_expect / mmd_grad; §3.2) ---------
def mmd_dense(st, q, sigmas):
    """Dense restatement of the squared MMD: L_b = d_bᵀ K d_b with d_b = |ψ_b|² − q and
    K(x,y) = Σ_σ exp(−(x−y)²/(2σ²)) ("radial-basis mixture over integer
    distance", DESIGN DECISIONS of SPEC §AD).  Returns (L[B], seed φ̄ = ∂L/∂ψ* = 2(Kd)⊙ψ).
    O(4^n): small n only."""
    st = np.ascontiguousarray(st, dtype=np.complex128)
    N = st.shape[1]
    x = np.arange(N, dtype=np.float64)
    d2 = (x[:, None] - x[None, :]) ** 2
    K = sum(np.exp(-d2 / (2.0 * s * s)) for s in np.atleast_1d(sigmas))
    d = np.abs(st) ** 2 - np.asarray(q)[None, :]
    Kd = d @ K  # K symmetric
    L = np.einsum("bx,bx->b", d, Kd)
    return L, 2.0 * Kd * st


def mmd_grad_dense(orc, st, n, em, theta, q, sigmas):
    """Reverse-mode MMD gradient on the oracle: forward with the oracle's apply, dense seed,
    then the oracle's backward (uncompute + θ̄ accumulation)."""
    psi = orc.apply_program(st, n, em, theta)
    L, phi = mmd_dense(psi, q, sigmas)
    phi = np.ascontiguousarray(phi)
    g = np.zeros(max(1, len(theta)))
    orc.backward(psi, phi, n, em, theta, g)
    return L, g[: len(theta)]


# ---- time evolution ("e^{-iHt}|ψ> equals dense matrix exponential") -----------
def pauli_dense(terms, n):
    """Dense 2^n x 2^n matrix of Σ c i^{nY} X^x Z^z for the (coef, xmask, zmask) triples of
    blocks.pauli_terms (qubit 1 = bit 0; Y = iXZ), the convention of pauli_axpy in qbg_oracle.cpp:
    (P ψ)[i] = c i^{nY} (-1)^{|(i^x) & z|} ψ[i^x]."""
    N = 1 << n
    H = np.zeros((N, N), dtype=np.complex128)
    idx = np.arange(N)
    for c, x, z in terms:
        ny = bin(int(x) & int(z)).count("1") & 3
        j = idx ^ int(x)
        sign = 1 - 2 * (np.array([bin(int(v) & int(z)).count("1") for v in j]) & 1)
        H[idx, j] += complex(c) * (1j ** ny) * sign
    return H


def expm_apply(st, terms, n, t):
    """e^{-iHt} applied to every batch row of st (dense scipy expm: small n only)."""
    import scipy.linalg
    U = scipy.linalg.expm(-1j * t * pauli_dense(terms, n))
    return (U @ np.asarray(st, dtype=np.complex128).T).T
