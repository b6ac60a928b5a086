"""Gate-matrix descriptors (the MatrixRepr classes, matrix.hpp:41-129) and the builtin gate
table (gates.hpp:32-94).  Pure host data; they cross the C-ABI as ``qbg_matrix`` / program
payloads.  Little-endian: matrix qubit 1 is the least significant bit."""
from __future__ import annotations

import cmath
import math

import numpy as np

from . import errors
from ._capi import MAT_DENSE, MAT_DIAGONAL, MAT_IDENTITY, MAT_PERMUTATION


class Matrix:
    kind: int
    dim: int

    def dense(self) -> np.ndarray:  # to_dense, matrix.hpp:229-233
        raise NotImplementedError

    def adjoint(self) -> "Matrix":  # adjoint_mat, matrix.hpp:594-643
        raise NotImplementedError


class Identity(Matrix):
    kind = MAT_IDENTITY

    def __init__(self, dim: int):
        if dim <= 0:
            raise errors.ShapeError("Identity: dimension must be positive")
        self.dim = dim

    def dense(self):
        return np.eye(self.dim, dtype=complex)

    def adjoint(self):
        return self


class Diagonal(Matrix):
    kind = MAT_DIAGONAL

    def __init__(self, diag):
        self.diag = np.asarray(diag, dtype=complex)
        if self.diag.size == 0:
            raise errors.ShapeError("Diagonal: dimension must be positive")
        self.dim = self.diag.size

    def dense(self):
        return np.diag(self.diag)

    def adjoint(self):
        return Diagonal(np.conj(self.diag))


class Permutation(Matrix):
    """Row i holds vals[i] at column perm[i] (matrix.hpp:56-58)."""

    kind = MAT_PERMUTATION

    def __init__(self, perm, vals):
        self.perm = np.asarray(perm, dtype=np.int64)
        self.vals = np.asarray(vals, dtype=complex)
        if self.perm.size == 0 or self.perm.size != self.vals.size:
            raise errors.ShapeError("Permutation: perm and vals must be non-empty and equal length")
        if sorted(self.perm.tolist()) != list(range(self.perm.size)):
            raise errors.ValidationError("Permutation: column indices must form a permutation")
        self.dim = self.perm.size

    def dense(self):
        m = np.zeros((self.dim, self.dim), dtype=complex)
        m[np.arange(self.dim), self.perm] = self.vals
        return m

    def adjoint(self):
        perm = np.empty_like(self.perm)
        vals = np.empty_like(self.vals)
        perm[self.perm] = np.arange(self.dim)
        vals[self.perm] = np.conj(self.vals)
        return Permutation(perm, vals)


class Dense(Matrix):
    """Square matrix; ``a[r, c]`` (stored column-major at the boundary, matrix.hpp:104)."""

    kind = MAT_DENSE

    def __init__(self, a):
        self.a = np.asarray(a, dtype=complex)
        if self.a.ndim != 2 or self.a.shape[0] != self.a.shape[1] or self.a.shape[0] == 0:
            raise errors.ShapeError("Dense: data size must be dim^2")
        self.dim = self.a.shape[0]

    def dense(self):
        return self.a.copy()

    def adjoint(self):
        return Dense(self.a.conj().T)


def payload(m: Matrix) -> tuple[np.ndarray, np.ndarray | None]:
    """Interleaved complex payload (+ permutation) in the C-ABI order."""
    if isinstance(m, Identity):
        return np.zeros(0, dtype=complex), None
    if isinstance(m, Diagonal):
        return m.diag, None
    if isinstance(m, Permutation):
        return m.vals, m.perm
    return np.ascontiguousarray(m.a.T).reshape(-1), None  # column-major


def as_matrix(m) -> Matrix:
    if isinstance(m, Matrix):
        return m
    return Dense(np.asarray(m, dtype=complex))


# ---- gate table, gates.hpp:32-94 ---------------------------------------------------------------
I1 = 1j
_S = 1.0 / math.sqrt(2.0)


def x():
    return Permutation([1, 0], [1.0, 1.0])


def y():
    return Permutation([1, 0], [-I1, I1])


def z():
    return Diagonal([1.0, -1.0])


def h():
    return Dense([[_S, _S], [_S, -_S]])


def i2():
    return Identity(2)


def s():
    return Diagonal([1.0, I1])


def sdag():
    return Diagonal([1.0, -I1])


def t():
    return Diagonal([1.0, cmath.rect(1.0, math.pi / 4)])


def tdag():
    return Diagonal([1.0, cmath.rect(1.0, -math.pi / 4)])


def swap():
    return Permutation([0, 2, 1, 3], [1, 1, 1, 1])


def cnot():  # control on qubit 2, X on qubit 1
    return Permutation([0, 1, 3, 2], [1, 1, 1, 1])


def cz():
    return Permutation([0, 1, 2, 3], [1, 1, 1, -1])


def toffoli():
    return Permutation([0, 1, 2, 3, 4, 5, 7, 6], [1] * 8)


def p0():
    return Dense([[1, 0], [0, 0]])


def p1():
    return Dense([[0, 0], [0, 1]])


def pu():
    return Dense([[0, 1], [0, 0]])


def pd():
    return Dense([[0, 0], [1, 0]])


def rx(theta):
    c, sn = math.cos(theta / 2), math.sin(theta / 2)
    return Dense([[c, -1j * sn], [-1j * sn, c]])


def ry(theta):
    c, sn = math.cos(theta / 2), math.sin(theta / 2)
    return Dense([[c, -sn], [sn, c]])


def rz(theta):
    return Diagonal([cmath.rect(1.0, -theta / 2), cmath.rect(1.0, theta / 2)])


def shift(theta):
    return Diagonal([1.0, cmath.rect(1.0, theta)])


def global_phase(theta, dim=2):
    return Diagonal([cmath.rect(1.0, theta)] * dim)


CONST_GATES = {
    "X": x, "Y": y, "Z": z, "H": h, "I2": i2, "S": s, "Sdag": sdag, "T": t, "Tdag": tdag,
    "SWAP": swap, "CNOT": cnot, "CZ": cz, "Toffoli": toffoli, "P0": p0, "P1": p1, "Pu": pu, "Pd": pd,
}
