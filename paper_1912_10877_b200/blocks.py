"""QBIR blocks and their lowering to device gate programs.

The block tree is host data.  ``apply(reg, block)`` walks it depth-first exactly like the
SPEC's dispatch (Chain left to right; Put/Kron/Repeat become instruct on
their locations; Control adds control masks) but instead of one C call per primitive it
emits a flat ``qbg_op`` program, compiled once by the engine (fusion plan + device payloads)
and re-parameterised by ``dispatch``.  Parameter order is the depth-first walk with shared
nodes contributing once."""
from __future__ import annotations

import ctypes
import math
from typing import Iterable, Sequence

import numpy as np

from . import errors
from . import matrix as M
from ._capi import (GEN_NONE, GEN_PHASE, GEN_ROTATION, GEN_SHIFT, MAX_CTRLS, MAX_TARGETS, QbgOp, QbgPauliTerm,
                    check, lib)


# ---------------------------------------------------------------------------------------------------
# block kinds
# ---------------------------------------------------------------------------------------------------
class Block:
    nqubits: int = 0

    def subblocks(self) -> list["Block"]:
        return []

    def __mul__(self, other):
        if isinstance(other, Block):  # matrix-product order: (A*B)|ψ> = A(B|ψ>)
            return Chain(self.nqubits, [other, self])
        return Scale(complex(other), self)

    def __rmul__(self, other):
        return Scale(complex(other), self)

    def __add__(self, other):
        return Add([self, other])

    def __neg__(self):
        return Scale(-1.0, self)

    @property
    def H(self):  # adjoint, Yao's `'`
        return dagger(self)


class Primitive(Block):
    pass


class ConstantGate(Primitive):
    def __init__(self, name: str, mat: M.Matrix):
        self.name = name
        self.mat = mat
        self.nqubits = int(round(math.log2(mat.dim)))

    def __repr__(self):
        return self.name


class Rotation(Primitive):
    """e^{-iΣθ/2} = cos(θ/2) I − i sin(θ/2) Σ for a reflexive generator Σ (gates.hpp:77-92)."""

    def __init__(self, generator: Block, theta: float):
        self.generator = generator
        self.theta = float(theta)
        self.nqubits = generator.nqubits

    def __repr__(self):
        return f"rot({self.generator!r}, {self.theta})"


class Shift(Primitive):
    """diag(1, e^{iθ}) (gates.hpp:72)."""

    nqubits = 1

    def __init__(self, theta: float):
        self.theta = float(theta)

    def __repr__(self):
        return f"shift({self.theta})"


class Phase(Primitive):
    """e^{iθ}·I (gates.hpp:73-75)."""

    nqubits = 1

    def __init__(self, theta: float):
        self.theta = float(theta)

    def __repr__(self):
        return f"phase({self.theta})"


class TimeEvolution(Primitive):
    """e^{-iHt} for a hermitian Pauli-sum H (Listing 6 ``time_evolve``).  The
    evolution time is the node's parameter (``theta``); applied on the device by a Krylov
    (Lanczos) exponential, ``qbg_time_evolve``."""

    def __init__(self, hamiltonian: Block, t: float):
        self.hamiltonian = hamiltonian
        self.theta = float(t)
        self.nqubits = hamiltonian.nqubits

    @property
    def t(self) -> float:
        return self.theta

    def __repr__(self):
        return f"time_evolve({self.hamiltonian!r}, {self.theta})"


class GeneralMatrix(Primitive):
    def __init__(self, mat):
        self.mat = M.as_matrix(mat)
        self.nqubits = int(round(math.log2(self.mat.dim)))


class Composite(Block):
    pass


class Chain(Composite):
    def __init__(self, n: int, blocks: Sequence[Block]):
        self.nqubits = n
        self.blocks = list(blocks)
        for b in self.blocks:
            if b.nqubits != n:
                raise errors.ShapeError(f"chain: child has {b.nqubits} qubits, expected {n}")

    def subblocks(self):
        return self.blocks


class Put(Composite):
    def __init__(self, n: int, locs: Sequence[int], block: Block):
        self.nqubits = n
        self.locs = tuple(int(l) for l in locs)
        self.block = block
        _check_locs(n, self.locs, "put")
        if len(self.locs) != block.nqubits:
            raise errors.ShapeError("put: location count differs from the block's qubit count")

    def subblocks(self):
        return [self.block]


class Control(Composite):
    def __init__(self, n: int, ctrl_locs: Sequence[int], ctrl_config: Sequence[int], locs: Sequence[int],
                 block: Block):
        self.nqubits = n
        self.ctrl_locs = tuple(int(c) for c in ctrl_locs)
        self.ctrl_config = tuple(int(c) for c in ctrl_config)
        self.locs = tuple(int(l) for l in locs)
        self.block = block
        _check_locs(n, self.locs + self.ctrl_locs, "control")
        if len(self.locs) != block.nqubits:
            raise errors.ShapeError("control: location count differs from the block's qubit count")

    def subblocks(self):
        return [self.block]


class Kron(Composite):
    def __init__(self, n: int, pairs: Sequence[tuple[tuple[int, ...], Block]]):
        self.nqubits = n
        self.pairs = [(tuple(l), b) for l, b in pairs]
        _check_locs(n, sum((l for l, _ in self.pairs), ()), "kron")

    def subblocks(self):
        return [b for _, b in self.pairs]


class Repeat(Composite):
    def __init__(self, n: int, block: Block, locs: Sequence[int]):
        self.nqubits = n
        self.block = block
        self.locs = tuple(int(l) for l in locs)
        _check_locs(n, self.locs, "repeat")

    def subblocks(self):
        return [self.block]


class Subroutine(Composite):
    """Subroutine (Listing 16): focus(locs) -> apply the child -> relax, i.e. the
    child on a local scope.  For a unitary child that is put(n, locs => child), and it lowers so
    (one program, fusable); a non-circuit child (Add / Scale) runs the explicit focus / relax."""

    def __init__(self, n: int, block: Block, locs: Sequence[int]):
        self.nqubits = n
        self.block = block
        self.locs = tuple(int(l) for l in locs)
        _check_locs(n, self.locs, "subroutine")
        if len(self.locs) != block.nqubits:
            raise errors.ShapeError("subroutine: location count differs from the block's qubit count")

    def subblocks(self):
        return [self.block]


class Add(Composite):
    def __init__(self, blocks: Sequence[Block]):
        self.blocks = []
        for b in blocks:  # flatten nested sums
            self.blocks.extend(b.blocks if isinstance(b, Add) else [b])
        if not self.blocks:
            raise errors.ValidationError("Add: needs at least one child")
        self.nqubits = self.blocks[0].nqubits

    def subblocks(self):
        return self.blocks


class Scale(Composite):
    def __init__(self, factor: complex, block: Block):
        self.factor = complex(factor)
        self.block = block
        self.nqubits = block.nqubits

    def subblocks(self):
        return [self.block]


class Cached(Composite):
    """cache(b) (Listings 6-7): transparent — apply through it equals apply
    without it.  The engine already keeps Pauli-sum operators as device programs."""

    def __init__(self, block: Block):
        self.block = block
        self.nqubits = block.nqubits

    def subblocks(self):
        return [self.block]


class Daggered(Composite):
    def __init__(self, block: Block):
        self.block = block
        self.nqubits = block.nqubits

    def subblocks(self):
        return [self.block]


def _check_locs(n, locs, what):
    if len(set(locs)) != len(locs):
        raise errors.ValidationError(f"{what}: duplicate location")
    for l in locs:
        if l < 1 or l > n:
            raise errors.RangeError(f"{what}: location out of range")


# ---------------------------------------------------------------------------------------------------
# constructors (Yao names)
# ---------------------------------------------------------------------------------------------------
X = ConstantGate("X", M.x())
Y = ConstantGate("Y", M.y())
Z = ConstantGate("Z", M.z())
H = ConstantGate("H", M.h())
I2 = ConstantGate("I2", M.i2())
S = ConstantGate("S", M.s())
Sdag = ConstantGate("Sdag", M.sdag())
T = ConstantGate("T", M.t())
Tdag = ConstantGate("Tdag", M.tdag())
SWAP = ConstantGate("SWAP", M.swap())
CNOT = ConstantGate("CNOT", M.cnot())
CZ = ConstantGate("CZ", M.cz())
Toffoli = ConstantGate("Toffoli", M.toffoli())
P0 = ConstantGate("P0", M.p0())
P1 = ConstantGate("P1", M.p1())
Pu = ConstantGate("Pu", M.pu())
Pd = ConstantGate("Pd", M.pd())
_HERMITIAN = {"X", "Y", "Z", "H", "I2", "SWAP", "CNOT", "CZ", "Toffoli", "P0", "P1"}
_PAIRS = {"S": "Sdag", "Sdag": "S", "T": "Tdag", "Tdag": "T", "Pu": "Pd", "Pd": "Pu"}
_CONSTS = {g.name: g for g in (X, Y, Z, H, I2, S, Sdag, T, Tdag, SWAP, CNOT, CZ, Toffoli, P0, P1, Pu, Pd)}


def define_const_gate(name: str, mat) -> ConstantGate:
    """gates.hpp:136-147"""
    m = M.as_matrix(mat)
    if m.dim < 2 or (m.dim & (m.dim - 1)):
        raise errors.ValidationError(f"define_const_gate: dimension must be a power of 2, got {m.dim}")
    g = ConstantGate(name, m)
    _CONSTS[name] = g
    return g


def Rx(theta):
    return Rotation(X, theta)


def Ry(theta):
    return Rotation(Y, theta)


def Rz(theta):
    return Rotation(Z, theta)


def rot(generator: Block, theta):
    return Rotation(generator, theta)


def shift(theta):
    return Shift(theta)


def phase(theta):
    return Phase(theta)


def matblock(m):
    return GeneralMatrix(m)


def time_evolve(h: Block, t: float) -> TimeEvolution:
    """time_evolve(h, t).  A Pauli expression is applied as a device Pauli sum;
    any other hermitian block through its sparse matrix (the Cached path, built once from mat(h))."""
    if not is_pauli_expression(h) and (h.nqubits > 16 or isinstance(h, TimeEvolution)):
        raise errors.UnsupportedError("time_evolve: h must be a Pauli expression or a small (n <= 16) block")
    return TimeEvolution(h, t)


def is_pauli_expression(b: Block) -> bool:
    try:
        pauli_terms(b)
        return True
    except errors.UnsupportedError:
        return False


def cache(b: Block) -> Cached:
    return Cached(b)


def _locs(l) -> tuple[int, ...]:
    return (int(l),) if isinstance(l, (int, np.integer)) else tuple(int(v) for v in l)


def chain(*args) -> Chain:
    """chain(n, b1, b2, ...) or chain(b1, b2, ...) (n inferred)."""
    if args and isinstance(args[0], (int, np.integer)):
        n, blocks = int(args[0]), args[1:]
    else:
        blocks = args
        n = blocks[0].nqubits
    if len(blocks) == 1 and isinstance(blocks[0], (list, tuple)):
        blocks = blocks[0]
    return Chain(n, list(blocks))


def put(n: int, locs, block: Block) -> Put:
    return Put(n, _locs(locs), block)


def control(n: int, ctrl_locs, locs, block: Block) -> Control:
    """Yao's control(n, ctrl, locs=>block); a negative control location is an inverse
    control (configuration 0)."""
    c = _locs(ctrl_locs)
    return Control(n, tuple(abs(v) for v in c), tuple(0 if v < 0 else 1 for v in c), _locs(locs), block)


def kron(*args) -> Kron:
    """kron(n, (loc, blk), ...) or kron(b1, b2, ...) on consecutive qubits."""
    if args and isinstance(args[0], (int, np.integer)):
        n = int(args[0])
        return Kron(n, [(_locs(l), b) for l, b in args[1:]])
    pairs, q = [], 1
    for b in args:
        pairs.append((tuple(range(q, q + b.nqubits)), b))
        q += b.nqubits
    return Kron(q - 1, pairs)


def repeat(n: int, block: Block, locs=None) -> Repeat:
    return Repeat(n, block, range(1, n + 1) if locs is None else _locs(locs))


def subroutine(n: int, block: Block, locs) -> Subroutine:
    return Subroutine(n, block, _locs(locs))


# ---------------------------------------------------------------------------------------------------
# parameters / dispatch / gatecount / dagger
# ---------------------------------------------------------------------------------------------------
def _param_nodes(b: Block, seen: dict, out: list):
    if isinstance(b, (Rotation, Shift, Phase, TimeEvolution)):
        if id(b) not in seen:
            seen[id(b)] = len(out)
            out.append(b)
        return
    for c in b.subblocks():
        _param_nodes(c, seen, out)


def parameter_nodes(b: Block) -> list[Block]:
    """Depth-first distinct parameterised nodes.  Block structure is immutable (only θ values
    change), so the list is cached on the block."""
    out = getattr(b, "_qbg_param_nodes", None)
    if out is None:
        out = []
        _param_nodes(b, {}, out)
        try:
            b._qbg_param_nodes = out
        except AttributeError:
            pass
    return out


def parameters(b: Block) -> np.ndarray:
    """Depth-first, each distinct node once."""
    return np.array([p.theta for p in parameter_nodes(b)], dtype=float)


def nparameters(b: Block) -> int:
    return len(parameter_nodes(b))


def dispatch(b: Block, arg, vec=None, rng=None) -> Block:
    """dispatch(b, vec) | dispatch(b, "random", rng=Rng(42)) | dispatch(b, op, vec) with
    θ ← op(θ, v) (Listing 9's ``dispatch!(-, circuit, lr*grad)``)."""
    nodes = parameter_nodes(b)
    if isinstance(arg, str) and arg == "random":
        from .register import Rng
        r = rng if rng is not None else Rng(42)
        for p in nodes:
            p.theta = r.uniform(0.0, 2 * math.pi)
        return b
    if callable(arg):
        v = np.asarray(vec, dtype=float)
        if v.size != len(nodes):
            raise errors.ValidationError("dispatch: parameter count mismatch")
        for p, x in zip(nodes, v):
            p.theta = float(arg(p.theta, x))
        return b
    v = np.asarray(arg, dtype=float).reshape(-1)
    if v.size != len(nodes):
        raise errors.ValidationError("dispatch: parameter count mismatch")
    for p, x in zip(nodes, v):
        p.theta = float(x)
    return b


def _gate_name(b: Block) -> str:
    if isinstance(b, ConstantGate):
        return b.name
    if isinstance(b, Rotation):
        g = b.generator
        if isinstance(g, ConstantGate) and g.name in ("X", "Y", "Z"):
            return "R" + g.name.lower()
        return "rot"
    if isinstance(b, Shift):
        return "shift"
    if isinstance(b, Phase):
        return "phase"
    return "matrix"


def gatecount(b: Block, _out=None, _ctrl=False) -> dict:
    """Histogram of primitive occurrences (shared nodes counted per occurrence).  Controlled
    primitives are keyed ``Control{<name>}``."""
    out = {} if _out is None else _out
    if isinstance(b, Primitive):
        k = f"Control{{{_gate_name(b)}}}" if _ctrl else _gate_name(b)
        out[k] = out.get(k, 0) + 1
        return out
    if isinstance(b, Control):
        gatecount(b.block, out, True)
        return out
    if isinstance(b, Repeat):
        for _ in b.locs:
            gatecount(b.block, out, _ctrl)
        return out
    for c in b.subblocks():
        gatecount(c, out, _ctrl)
    return out


def dagger(b: Block) -> Block:
    """adjoint_block."""
    if isinstance(b, ConstantGate):
        if b.name in _HERMITIAN:
            return b
        if b.name in _PAIRS:
            return _CONSTS[_PAIRS[b.name]]
        return GeneralMatrix(b.mat.adjoint())
    if isinstance(b, Rotation):
        return Rotation(b.generator, -b.theta)
    if isinstance(b, Shift):
        return Shift(-b.theta)
    if isinstance(b, Phase):
        return Phase(-b.theta)
    if isinstance(b, GeneralMatrix):
        return GeneralMatrix(b.mat.adjoint())
    if isinstance(b, TimeEvolution):
        return TimeEvolution(b.hamiltonian, -b.theta)
    if isinstance(b, Cached):
        return Cached(dagger(b.block))
    if isinstance(b, Chain):
        return Chain(b.nqubits, [dagger(c) for c in reversed(b.blocks)])
    if isinstance(b, Put):
        return Put(b.nqubits, b.locs, dagger(b.block))
    if isinstance(b, Control):
        return Control(b.nqubits, b.ctrl_locs, b.ctrl_config, b.locs, dagger(b.block))
    if isinstance(b, Kron):
        return Kron(b.nqubits, [(l, dagger(c)) for l, c in b.pairs])
    if isinstance(b, Repeat):
        return Repeat(b.nqubits, dagger(b.block), b.locs)
    if isinstance(b, Subroutine):
        return Subroutine(b.nqubits, dagger(b.block), b.locs)
    if isinstance(b, Scale):
        return Scale(b.factor.conjugate(), dagger(b.block))
    if isinstance(b, Add):
        return Add([dagger(c) for c in b.blocks])
    if isinstance(b, Daggered):
        return b.block
    return Daggered(b)


# ---------------------------------------------------------------------------------------------------
# matrices (host algebra; small sizes only — used for generators and by tests)
# ---------------------------------------------------------------------------------------------------
def _embed(n: int, locs: Sequence[int], m: np.ndarray, ctrls=(), cfg=()) -> np.ndarray:
    """Dense 2^n operator of m on locs (matrix qubit q -> locs[q]) with control projectors."""
    dim = 1 << n
    t = len(locs)
    out = np.zeros((dim, dim), dtype=complex)
    for col in range(dim):
        if any(((col >> (c - 1)) & 1) != v for c, v in zip(ctrls, cfg)):
            out[col, col] += 1
            continue
        sub = sum(((col >> (l - 1)) & 1) << q for q, l in enumerate(locs))
        base = col
        for l in locs:
            base &= ~(1 << (l - 1))
        for r in range(1 << t):
            row = base
            for q, l in enumerate(locs):
                if (r >> q) & 1:
                    row |= 1 << (l - 1)
            out[row, col] += m[r, sub]
    return out


def mat(b: Block) -> np.ndarray:
    """Dense operator of a block (Chain multiplies in reverse order)."""
    n = b.nqubits
    if isinstance(b, ConstantGate) or isinstance(b, GeneralMatrix):
        return b.mat.dense()
    if isinstance(b, Rotation):
        g = mat(b.generator)
        c, s = math.cos(b.theta / 2), math.sin(b.theta / 2)
        return c * np.eye(g.shape[0]) - 1j * s * g
    if isinstance(b, Shift):
        return M.shift(b.theta).dense()
    if isinstance(b, Phase):
        return M.global_phase(b.theta).dense()
    if isinstance(b, Chain):
        out = np.eye(1 << n, dtype=complex)
        for c in b.blocks:
            out = mat(c) @ out
        return out
    if isinstance(b, (Put, Subroutine)):
        return _embed(n, b.locs, mat(b.block))
    if isinstance(b, Control):
        return _embed(n, b.locs, mat(b.block), b.ctrl_locs, b.ctrl_config)
    if isinstance(b, Kron):
        out = np.eye(1 << n, dtype=complex)
        for l, c in b.pairs:
            out = _embed(n, l, mat(c)) @ out
        return out
    if isinstance(b, Repeat):
        out = np.eye(1 << n, dtype=complex)
        for l in b.locs:
            out = _embed(n, (l,), mat(b.block)) @ out
        return out
    if isinstance(b, Add):
        return sum(mat(c) for c in b.blocks)
    if isinstance(b, Scale):
        return b.factor * mat(b.block)
    if isinstance(b, Daggered):
        return mat(b.block).conj().T
    if isinstance(b, Cached):
        return mat(b.block)
    if isinstance(b, TimeEvolution):
        import scipy.linalg
        return scipy.linalg.expm(-1j * b.theta * mat(b.hamiltonian))
    raise errors.UnsupportedError(f"mat: unsupported block {type(b).__name__}")


def _class_matrix(b: Block) -> M.Matrix:
    """Matrix of a constant block in the most specific class (generator payloads)."""
    if isinstance(b, ConstantGate) or isinstance(b, GeneralMatrix):
        return b.mat
    d = mat(b)
    off = d - np.diag(np.diag(d))
    if not off.any():
        return M.Diagonal(np.diag(d))
    nz = d != 0
    if (nz.sum(axis=1) == 1).all() and (nz.sum(axis=0) == 1).all():
        perm = nz.argmax(axis=1)
        return M.Permutation(perm, d[np.arange(d.shape[0]), perm])
    return M.Dense(d)


# ---------------------------------------------------------------------------------------------------
# lowering to a device program
# ---------------------------------------------------------------------------------------------------
class _Emitter:
    def __init__(self, slots: dict):
        self.ops: list[QbgOp] = []
        self.vals: list[complex] = []
        self.perms: list[int] = []
        self.slots = slots

    def emit(self, kind_mat: M.Matrix | None, gen: int, param: int, targets, ctrls, cfg, dim: int):
        if len(targets) > MAX_TARGETS:
            raise errors.UnsupportedError("apply: primitive wider than 5 qubits")
        if len(ctrls) > MAX_CTRLS:
            raise errors.UnsupportedError("apply: more than 16 controls")
        op = QbgOp()
        op.gen, op.param, op.ntarget, op.nctrl, op.dim = gen, param, len(targets), len(ctrls), dim
        for k, t in enumerate(targets):
            op.targets[k] = t
        for k, (c, v) in enumerate(zip(ctrls, cfg)):
            op.ctrls[k] = c
            op.ctrl_cfg[k] = v
        if kind_mat is None:
            op.kind = M.MAT_DIAGONAL
            op.data = 0
            op.perm = 0
        else:
            op.kind = kind_mat.kind
            vals, perm = M.payload(kind_mat)
            op.data = len(self.vals)
            self.vals.extend(complex(v) for v in vals)
            op.perm = len(self.perms)
            if perm is not None:
                self.perms.extend(int(p) for p in perm)
        self.ops.append(op)


def _lower(b: Block, qmap: tuple, ctrls: tuple, cfg: tuple, em: _Emitter, adjoint=False):
    if isinstance(b, ConstantGate) or isinstance(b, GeneralMatrix):
        m = b.mat.adjoint() if adjoint else b.mat
        em.emit(m, GEN_NONE, -1, qmap, ctrls, cfg, m.dim)
    elif isinstance(b, Rotation):
        if adjoint:
            raise errors.UnsupportedError("Daggered parameterised block: use dagger(block)")
        em.emit(_class_matrix(b.generator), GEN_ROTATION, em.slots[id(b)], qmap, ctrls, cfg, 1 << b.nqubits)
    elif isinstance(b, Shift):
        if adjoint:
            raise errors.UnsupportedError("Daggered parameterised block: use dagger(block)")
        em.emit(None, GEN_SHIFT, em.slots[id(b)], qmap, ctrls, cfg, 2)
    elif isinstance(b, Phase):
        if adjoint:
            raise errors.UnsupportedError("Daggered parameterised block: use dagger(block)")
        em.emit(None, GEN_PHASE, em.slots[id(b)], qmap, ctrls, cfg, 1 << b.nqubits)
    elif isinstance(b, Chain):
        seq = reversed(b.blocks) if adjoint else b.blocks
        for c in seq:
            _lower(c, qmap, ctrls, cfg, em, adjoint)
    elif isinstance(b, (Put, Subroutine)):
        _lower(b.block, tuple(qmap[l - 1] for l in b.locs), ctrls, cfg, em, adjoint)
    elif isinstance(b, Control):
        _lower(b.block, tuple(qmap[l - 1] for l in b.locs), ctrls + tuple(qmap[c - 1] for c in b.ctrl_locs),
               cfg + b.ctrl_config, em, adjoint)
    elif isinstance(b, Kron):
        for l, c in (reversed(b.pairs) if adjoint else b.pairs):
            _lower(c, tuple(qmap[v - 1] for v in l), ctrls, cfg, em, adjoint)
    elif isinstance(b, Repeat):
        for l in (reversed(b.locs) if adjoint else b.locs):
            _lower(b.block, (qmap[l - 1],), ctrls, cfg, em, adjoint)
    elif isinstance(b, Daggered):
        _lower(b.block, qmap, ctrls, cfg, em, not adjoint)
    elif isinstance(b, Cached):
        _lower(b.block, qmap, ctrls, cfg, em, adjoint)
    elif isinstance(b, TimeEvolution):
        raise errors.UnsupportedError("time_evolve: not a gate program (applied by the Krylov engine)")
    else:
        raise errors.UnsupportedError(f"apply: {type(b).__name__} is not a circuit block (non-unitary)")


class Program:
    """A compiled gate program (``qbg_prog``): the lowering of one block tree."""

    def __init__(self, block: Block):
        self.block = block
        nodes = parameter_nodes(block)
        slots = {id(p): k for k, p in enumerate(nodes)}
        em = _Emitter(slots)
        n = block.nqubits
        _lower(block, tuple(range(1, n + 1)), (), (), em)
        self.nparams = len(nodes)
        self.nops = len(em.ops)
        ops = (QbgOp * max(1, len(em.ops)))(*em.ops)
        vals = np.ascontiguousarray(np.array(em.vals or [0j], dtype=np.complex128))
        perms = np.ascontiguousarray(np.array(em.perms or [0], dtype=np.int64))
        h = ctypes.c_void_p()
        check(lib().qbg_prog_create(n, ops, len(em.ops), vals.ctypes.data, len(em.vals), perms.ctypes.data,
                                    len(em.perms), ctypes.byref(h)))
        self._h = h
        self._theta = None
        self.sync_params()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().qbg_prog_destroy(h)
            self._h = None

    def sync_params(self, theta=None):
        th = parameters(self.block) if theta is None else np.asarray(theta, dtype=float)
        if self._theta is not None and np.array_equal(th, self._theta):
            return
        th = np.ascontiguousarray(th, dtype=np.float64)
        check(lib().qbg_prog_set_params(self._h, th.ctypes.data if th.size else None, th.size))
        self._theta = th.copy()

    def stats(self) -> dict:
        f, b, g = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib().qbg_prog_stats(self._h, ctypes.byref(f), ctypes.byref(b), ctypes.byref(g)))
        return {"fwd_passes": f.value, "bwd_passes": b.value, "gates": g.value}

    def plan_info(self) -> str:
        """Fusion plans built so far (passes, tile qubits, stages, ops per stage)."""
        buf = ctypes.create_string_buffer(1 << 20)
        check(lib().qbg_prog_plan_info(self._h, buf, len(buf)))
        return buf.value.decode()

    def plan_preview(self, nbatch: int = 1, dtype: str = "c128") -> str:
        """Runs the fusion planner on the host only (no GPU needed)."""
        buf = ctypes.create_string_buffer(1 << 20)
        check(lib().qbg_prog_plan_preview(self._h, nbatch, 0 if dtype == "c128" else 1, buf, len(buf)))
        return buf.value.decode()

    # raw op list (for the oracle / tests)
    def lowered(self):
        nodes = parameter_nodes(self.block)
        em = _Emitter({id(p): k for k, p in enumerate(nodes)})
        _lower(self.block, tuple(range(1, self.block.nqubits + 1)), (), (), em)
        return em


_PROGRAMS: dict[int, Program] = {}


def compile_block(b: Block) -> Program:
    """Compiled program for a block, cached on the block object (structure is immutable;
    parameters are re-synchronised on every use)."""
    p = getattr(b, "_qbg_program", None)
    if p is None:
        p = Program(b)
        b._qbg_program = p
    p.sync_params()
    return p


def apply(reg, b: Block):
    """apply!(reg, block), in place.  Add/Scale (observables) are applied
    as linear maps on clones (≤ 2 live scratch states)."""
    if b.nqubits != reg.nactive:
        raise errors.ShapeError("apply: block qubit count differs from active qubits")
    if isinstance(b, Scale):
        apply(reg, b.block)
        return reg.scale(b.factor)
    if isinstance(b, Subroutine) and not is_circuit(b):
        na = reg.nactive
        reg.focus(*b.locs)
        apply(reg, b.block)
        return reg.relax(*b.locs, to_nactive=na)
    if isinstance(b, Add):
        src = reg.copy()
        first = True
        for c in b.blocks:
            tmp = src.copy()
            apply(tmp, c)
            if first:
                reg.assign(tmp)
                first = False
            else:
                reg.add_scaled(tmp, 1.0)
        return reg
    if has_time_evolution(b):
        for kind, seg in segments(b):
            if kind == "te":
                evolve(reg, seg.hamiltonian, seg.theta)
            else:
                check(lib().qbg_apply(reg._h, compile_block(seg)._h))
        return reg
    p = compile_block(b)
    check(lib().qbg_apply(reg._h, p._h))
    return reg


def is_circuit(b: Block) -> bool:
    """No Add / Scale anywhere: the block lowers to one gate program."""
    if isinstance(b, (Add, Scale)):
        return False
    return all(is_circuit(c) for c in b.subblocks())


# ---------------------------------------------------------------------------------------------------
# time evolution inside circuits: the circuit splits into gate-program segments and Krylov steps
# ---------------------------------------------------------------------------------------------------
def has_time_evolution(b: Block) -> bool:
    v = getattr(b, "_qbg_has_te", None)
    if v is None:
        v = isinstance(b, TimeEvolution) or any(has_time_evolution(c) for c in b.subblocks())
        try:
            b._qbg_has_te = v
        except AttributeError:
            pass
    return v


def segments(b: Block) -> list:
    """[("prog", chain) | ("te", TimeEvolution)] in application order, cached on the block (its
    structure is immutable).  TimeEvolution may appear at the top level of (nested) chains and
    inside cache(); under put / control / kron it is unsupported."""
    segs = getattr(b, "_qbg_segments", None)
    if segs is not None:
        return segs
    flat: list = []

    def walk(x):
        if isinstance(x, TimeEvolution):
            flat.append(x)
        elif isinstance(x, Cached):
            walk(x.block)
        elif isinstance(x, Chain) and has_time_evolution(x):
            for c in x.blocks:
                walk(c)
        elif has_time_evolution(x):
            raise errors.UnsupportedError("time_evolve: only inside chains (not under put / control / kron)")
        else:
            flat.append(x)

    walk(b)
    segs, run = [], []
    for x in flat:
        if isinstance(x, TimeEvolution):
            if run:
                segs.append(("prog", Chain(b.nqubits, run)))
                run = []
            segs.append(("te", x))
        else:
            run.append(x)
    if run:
        segs.append(("prog", Chain(b.nqubits, run)))
    b._qbg_segments = segs
    return segs


def evolve(reg, H: Block, t: float, tol: float = 1e-12, maxdim: int = 30) -> int:
    """|reg> <- e^{-iHt}|reg> on the device (qbg_time_evolve for a Pauli sum, qbg_time_evolve_sparse
    otherwise); returns the Krylov dimension used."""
    used = ctypes.c_int32()
    if is_pauli_expression(H):
        check(lib().qbg_time_evolve(reg._h, compile_observable(H)._h, float(t), float(tol), int(maxdim),
                                    ctypes.byref(used)))
    else:
        check(lib().qbg_time_evolve_sparse(reg._h, sparse_operator(H)._h, float(t), float(tol), int(maxdim),
                                           ctypes.byref(used)))
    return used.value


def apply_hamiltonian(H: Block, reg, out=None):
    """out = H|reg> (Pauli sum or sparse operator), on the device."""
    from .register import Register
    if out is None:
        out = Register(reg.nqubits, reg.nbatch, dtype=reg.dtype)
    if is_pauli_expression(H):
        check(lib().qbg_obs_apply(reg._h, compile_observable(H)._h, out._h))
    else:
        check(lib().qbg_sparse_apply(reg._h, sparse_operator(H)._h, out._h))
    return out


class SparseOperator:
    """A full-register sparse operator on the device (the reference's Cached matrix,
    SparseColumns + matvec_cols): built from a matrix (dense / scipy.sparse) of dimension 2^n."""

    def __init__(self, m):
        import scipy.sparse as sp
        a = sp.csc_matrix(m, dtype=np.complex128)
        a.sum_duplicates()
        a.sort_indices()
        d = a.shape[0]
        n = int(d).bit_length() - 1
        if a.shape != (d, d) or d != (1 << n):
            raise errors.ShapeError("sparse operator: matrix must be 2^n x 2^n")
        colptr = np.ascontiguousarray(a.indptr, dtype=np.int64)
        rows = np.ascontiguousarray(a.indices, dtype=np.int64)
        vals = np.ascontiguousarray(a.data, dtype=np.complex128)
        h = ctypes.c_void_p()
        check(lib().qbg_sparse_create(n, a.nnz, colptr.ctypes.data, rows.ctypes.data if a.nnz else None,
                                      vals.ctypes.data if a.nnz else None, ctypes.byref(h)))
        self._h, self.nqubits, self.nnz = h, n, a.nnz

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().qbg_sparse_destroy(h)
            except Exception:
                pass

    def apply(self, reg, out=None):
        from .register import Register
        if out is None:
            out = Register(reg.nqubits, reg.nbatch, dtype=reg.dtype)
        check(lib().qbg_sparse_apply(reg._h, self._h, out._h))
        return out


def sparse_operator(b: Block) -> SparseOperator:
    """The sparse operator of a block, built once from mat(b) and cached on the block."""
    op = getattr(b, "_qbg_sparse", None)
    if op is None:
        op = SparseOperator(mat(b))
        b._qbg_sparse = op
    return op


# ---------------------------------------------------------------------------------------------------
# observables: Add/Scale/Chain/Put/Kron/Repeat of Pauli primitives -> Pauli terms
# ---------------------------------------------------------------------------------------------------
_PAULI_XZ = {"I2": (0, 0), "X": (1, 0), "Y": (1, 1), "Z": (0, 1)}


def _pmul(a, b):
    """(c1, x1, z1)·(c2, x2, z2) for Pauli strings P = ⊗σ, σ from (x, z) bits with Y = (1, 1)."""
    c1, x1, z1 = a
    c2, x2, z2 = b
    # per qubit: σ(x1,z1)σ(x2,z2) = phase · σ(x1^x2, z1^z2)
    ph = 1 + 0j
    q = x1 | z1 | x2 | z2
    while q:
        bit = q & -q
        q ^= bit
        s1 = ((x1 & bit) != 0, (z1 & bit) != 0)
        s2 = ((x2 & bit) != 0, (z2 & bit) != 0)
        ph *= _SIGMA_PHASE[s1][s2]
    return (c1 * c2 * ph, x1 ^ x2, z1 ^ z2)


_I, _X, _Y, _Z = (False, False), (True, False), (True, True), (False, True)
_SIGMA_PHASE = {
    _I: {_I: 1, _X: 1, _Y: 1, _Z: 1},
    _X: {_I: 1, _X: 1, _Y: 1j, _Z: -1j},
    _Y: {_I: 1, _X: -1j, _Y: 1, _Z: 1j},
    _Z: {_I: 1, _X: 1j, _Y: -1j, _Z: 1},
}


def pauli_terms(b: Block, qmap=None) -> list[tuple[complex, int, int]]:
    n = b.nqubits
    qmap = tuple(range(1, n + 1)) if qmap is None else qmap
    if isinstance(b, ConstantGate) and b.name in _PAULI_XZ:
        x, z = _PAULI_XZ[b.name]
        if b.nqubits != 1:
            raise errors.UnsupportedError("observable: not a Pauli expression")
        bit = 1 << (qmap[0] - 1)
        return [(1 + 0j, bit if x else 0, bit if z else 0)]
    if isinstance(b, Add):
        return [t for c in b.blocks for t in pauli_terms(c, qmap)]
    if isinstance(b, Cached):
        return pauli_terms(b.block, qmap)
    if isinstance(b, Scale):
        return [(b.factor * c, x, z) for c, x, z in pauli_terms(b.block, qmap)]
    if isinstance(b, Put):
        return pauli_terms(b.block, tuple(qmap[l - 1] for l in b.locs))
    if isinstance(b, (Chain, Kron, Repeat)):
        if isinstance(b, Chain):
            parts = [pauli_terms(c, qmap) for c in b.blocks]
            parts = parts[::-1]  # operator product: later blocks multiply from the left
        elif isinstance(b, Kron):
            parts = [pauli_terms(c, tuple(qmap[v - 1] for v in l)) for l, c in b.pairs]
        else:
            parts = [pauli_terms(b.block, (qmap[l - 1],)) for l in b.locs]
        acc = [(1 + 0j, 0, 0)]
        for p in parts:
            acc = [_pmul(a, t) for a in acc for t in p]
        return acc
    raise errors.UnsupportedError(f"observable: {type(b).__name__} is not a Pauli expression")


class Observable:
    """A compiled Pauli-sum observable (``qbg_obs``)."""

    def __init__(self, block: Block):
        self.block = block
        terms = pauli_terms(block)
        self.nterms = len(terms)
        arr = (QbgPauliTerm * max(1, len(terms)))()
        for k, (c, x, z) in enumerate(terms):
            arr[k] = QbgPauliTerm(c.real, c.imag, x, z)
        self.terms = terms
        h = ctypes.c_void_p()
        check(lib().qbg_obs_create(block.nqubits, arr, len(terms), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().qbg_obs_destroy(h)
            self._h = None


def compile_observable(b: Block) -> Observable:
    o = getattr(b, "_qbg_obs", None)
    if o is None:
        o = Observable(b)
        b._qbg_obs = o
    return o
