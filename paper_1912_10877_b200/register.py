"""Device register and its instruction set — the host mirror of qblock's register module
(register.hpp:58-493) over the C-ABI.  A :class:`Register` owns a batch-innermost device
buffer; ``state()`` / ``set_state()`` move amplitudes in the reference's host layout
(batch slowest, shape ``(nbatch, 2**nqubits)``)."""
from __future__ import annotations

import ctypes
from typing import Iterable, Sequence

import numpy as np

from . import errors
from ._capi import QBG_C64, QBG_C128, QbgMatrix, check, i32, lib
from .matrix import Matrix, as_matrix, payload

DTYPES = {"c128": QBG_C128, "complex128": QBG_C128, "c64": QBG_C64, "complex64": QBG_C64}


class Rng:
    """qblock::Rng (rng.hpp:25-66): SplitMix64-mixed seed driving std::mt19937_64."""

    def __init__(self, seed: int = 42, _handle=None, _owned=True):
        self._owned = _owned
        if _handle is None:
            h = ctypes.c_void_p()
            check(lib().qbg_rng_create(seed, ctypes.byref(h)))
            _handle = h
        self._h = _handle

    def __del__(self):
        if getattr(self, "_owned", False) and self._h:
            lib().qbg_rng_destroy(self._h)
            self._h = None

    def split(self, label) -> "Rng":
        h = ctypes.c_void_p()
        if isinstance(label, str):
            check(lib().qbg_rng_split_label(self._h, label.encode(), ctypes.byref(h)))
        else:
            check(lib().qbg_rng_split_salt(self._h, int(label), ctypes.byref(h)))
        return Rng(_handle=h)

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        if lo is None:
            return lib().qbg_rng_uniform(self._h)
        return lib().qbg_rng_uniform_range(self._h, lo, hi)

    def gauss(self) -> float:
        return lib().qbg_rng_gauss(self._h)

    def bits(self) -> int:
        return lib().qbg_rng_bits(self._h)


def set_qubit_cap(n: int) -> None:
    """register.hpp:41"""
    check(lib().qbg_set_qubit_cap(n))


def qubit_cap() -> int:
    return lib().qbg_get_qubit_cap()


def state_alloc_counter() -> int:
    """register.hpp:45-48: number of full-state device allocations so far."""
    return lib().qbg_alloc_count()


class Register:
    """Register(nqubits, nbatch, seed), register.hpp:60-70."""

    def __init__(self, nqubits: int, nbatch: int = 1, seed: int = 42, dtype: str = "c128", _handle=None):
        if _handle is None:
            h = ctypes.c_void_p()
            check(lib().qbg_reg_create(nqubits, nbatch, DTYPES[dtype], seed, ctypes.byref(h)))
            _handle = h
        self._h = _handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().qbg_reg_destroy(h)
            self._h = None

    # ---- shape ---------------------------------------------------------------------------------
    def _info(self):
        nq, na, dt = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        nb = ctypes.c_int64()
        check(lib().qbg_reg_info(self._h, ctypes.byref(nq), ctypes.byref(na), ctypes.byref(nb), ctypes.byref(dt)))
        return nq.value, na.value, nb.value, dt.value

    @property
    def nqubits(self) -> int:
        return self._info()[0]

    @property
    def nactive(self) -> int:
        return self._info()[1]

    @property
    def nremain(self) -> int:
        nq, na, _, _ = self._info()
        return nq - na

    @property
    def nbatch(self) -> int:
        return self._info()[2]

    @property
    def dtype(self) -> str:
        return "c128" if self._info()[3] == QBG_C128 else "c64"

    @property
    def device_ptr(self) -> int:
        return lib().qbg_reg_device_ptr(self._h)

    @property
    def rng(self) -> Rng:
        return Rng(_handle=ctypes.c_void_p(lib().qbg_reg_rng(self._h)), _owned=False)

    def nbytes(self) -> int:
        nq, _, nb, dt = self._info()
        return (1 << nq) * nb * (16 if dt == QBG_C128 else 8)

    # ---- data movement (reference layout) ------------------------------------------------------------
    def state(self) -> np.ndarray:
        """Amplitudes, shape (nbatch, 2**nqubits), complex128 (Register::batch, 109-117)."""
        nq, _, nb, _ = self._info()
        out = np.empty((nb, 1 << nq), dtype=np.complex128)
        check(lib().qbg_download(self._h, out.ctypes.data, out.size))
        return out

    def set_state(self, amps) -> "Register":
        nq, _, nb, _ = self._info()
        a = np.ascontiguousarray(np.asarray(amps, dtype=np.complex128).reshape(nb, 1 << nq))
        check(lib().qbg_upload(self._h, a.ctypes.data, a.size))
        check(lib().qbg_synchronize())
        return self

    def copy(self) -> "Register":
        """Register(const Register&), register.hpp:72-80 (counts an allocation)."""
        h = ctypes.c_void_p()
        check(lib().qbg_reg_clone(self._h, ctypes.byref(h)))
        return Register(0, _handle=h)

    clone = copy

    def assign(self, other: "Register") -> "Register":
        check(lib().qbg_reg_copy(self._h, other._h))
        return self

    # ---- algebra (register.hpp:120-150) ------------------------------------------------------------------
    def norm(self, b: int | None = None):
        out = np.empty(self.nbatch)
        check(lib().qbg_norm(self._h, out.ctypes.data))
        return out if b is None else float(out[b])

    def inner(self, other: "Register") -> np.ndarray:
        out = np.empty(2 * self.nbatch)
        check(lib().qbg_inner(self._h, other._h, out.ctypes.data))
        return out[0::2] + 1j * out[1::2]

    def scale(self, factor: complex) -> "Register":
        f = complex(factor)
        check(lib().qbg_scale(self._h, f.real, f.imag))
        return self

    def add_scaled(self, other: "Register", factor: complex = 1.0) -> "Register":
        f = complex(factor)
        check(lib().qbg_add_scaled(self._h, other._h, f.real, f.imag))
        return self

    # ---- state files (register.hpp:181-205) -------------------------------------------------------------------
    def save(self, path: str) -> None:
        """QBREG1 file, interchangeable with qblock::Register::save."""
        check(lib().qbg_save(self._h, str(path).encode()))

    @staticmethod
    def load(path: str, seed: int = 42, dtype: str = "c128") -> "Register":
        h = ctypes.c_void_p()
        check(lib().qbg_load(str(path).encode(), seed, DTYPES[dtype], ctypes.byref(h)))
        return Register(0, _handle=h)

    # ---- focus / relax (register.hpp:156-177) ---------------------------------------------------------------
    def focus(self, *locs) -> "Register":
        arr, n = i32(_flat(locs))
        check(lib().qbg_focus(self._h, arr, n))
        return self

    def relax(self, *locs, to_nactive: int | None = None) -> "Register":
        arr, n = i32(_flat(locs))
        if to_nactive is None:
            to_nactive = self.nqubits
        check(lib().qbg_relax(self._h, arr, n, to_nactive))
        return self

    def __repr__(self):
        nq, na, nb, _ = self._info()
        return f"Register(nqubits={nq}, nactive={na}, nbatch={nb}, dtype={self.dtype})"


def _flat(locs) -> list[int]:
    if len(locs) == 1 and isinstance(locs[0], (tuple, list, range)):
        return [int(v) for v in locs[0]]
    return [int(v) for v in locs]


# ---- constructors (register.hpp:260-286) -------------------------------------------------------------------
def zero_state(n: int, nbatch: int = 1, seed: int = 42, dtype: str = "c128") -> Register:
    r = Register(n, nbatch, seed, dtype)
    check(lib().qbg_set_zero(r._h))
    return r


def rand_state(n: int, nbatch: int = 1, seed: int = 42, dtype: str = "c128") -> Register:
    r = Register(n, nbatch, seed, dtype)
    check(lib().qbg_set_rand(r._h, seed))
    return r


def product_state(bits, nbits: int | None = None, nbatch: int = 1, seed: int = 42, dtype: str = "c128") -> Register:
    """``bits``: an int (with ``nbits``), a '0101' string (qubit 1 rightmost, bits.hpp:126-139),
    or one int per batch."""
    if isinstance(bits, str):
        nbits = len(bits)
        vals = [int(bits, 2)]
    elif isinstance(bits, Iterable):
        vals = [int(b) for b in bits]
    else:
        vals = [int(bits)]
    if nbits is None:
        raise errors.ValidationError("product_state: nbits is required for integer bit strings")
    if len(vals) > 1:
        nbatch = len(vals)
    r = Register(nbits, nbatch, seed, dtype)
    arr = (ctypes.c_uint64 * len(vals))(*vals)
    check(lib().qbg_set_product(r._h, arr, len(vals)))
    return r


# ---- instruct (register.hpp:392-408) ---------------------------------------------------------------------------
def instruct(reg: Register, gate, locs: Sequence[int], ctrl_locs: Sequence[int] = (),
             ctrl_config: Sequence[int] = (), params: Sequence[float] = ()) -> Register:
    """``gate`` is a tag ("X", "Rx", ...) resolved by gate_by_tag (gates.hpp:156-175) or a
    :class:`~paper_1912_10877_b200.matrix.Matrix` / square array."""
    if isinstance(locs, int):
        locs = (locs,)
    if isinstance(ctrl_locs, int):
        ctrl_locs = (ctrl_locs,)
    if isinstance(ctrl_config, int):
        ctrl_config = (ctrl_config,)
    if len(ctrl_locs) != len(ctrl_config):
        raise errors.ValidationError("instruct: control locations and configuration differ in length")
    la, nl = i32(locs)
    ca, nc = i32(ctrl_locs)
    fa, _ = i32(ctrl_config)
    if isinstance(gate, str):
        p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(-1))
        pp = p.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if p.size else None
        check(lib().qbg_instruct_tag(reg._h, gate.encode(), la, nl, ca, fa, nc, pp, p.size))
        return reg
    m = as_matrix(gate)
    vals, perm = payload(m)
    vals = np.ascontiguousarray(vals, dtype=np.complex128)
    perm_arr = np.ascontiguousarray(perm if perm is not None else np.zeros(1, np.int64), dtype=np.int64)
    qm = QbgMatrix(m.kind, m.dim, vals.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                   perm_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    check(lib().qbg_instruct(reg._h, ctypes.byref(qm), la, nl, ca, fa, nc))
    return reg


# ---- measurement (register.hpp:414-493) -------------------------------------------------------------------------
def probabilities(reg: Register, b: int = 0) -> np.ndarray:
    out = np.empty(1 << reg.nactive)
    check(lib().qbg_probabilities(reg._h, b, out.ctypes.data))
    return out


def measure(reg: Register, nshots: int = 1, rng: Rng | None = None) -> np.ndarray:
    """Non-destructive sampling; returns basis indices, shape (nbatch, nshots) grouped by batch.
    Without ``rng`` the register's own stream is used (register.hpp:457-459)."""
    nb = reg.nbatch
    out = np.empty(nb * max(nshots, 1), dtype=np.uint64)
    check(lib().qbg_measure(reg._h, nshots, rng._h if rng is not None else None, out.ctypes.data))
    return out.reshape(nb, nshots)


def measure_collapse(reg: Register, rng: Rng | None = None) -> np.ndarray:
    """measure!: one sample per batch, collapsing each batch onto it (register.hpp:462-493)."""
    out = np.empty(reg.nbatch, dtype=np.uint64)
    check(lib().qbg_measure_collapse(reg._h, rng._h if rng is not None else None, out.ctypes.data))
    return out


def to_text(value: int, nbits: int) -> str:
    """bits.hpp:104-112: qubit 1 rightmost, '0010 (2)'."""
    return format(int(value), f"0{nbits}b") + " (2)"
