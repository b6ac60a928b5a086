"""paper_1912_10877_b200 — a B200-native (sm_100a) state-vector engine for Yao-style
differentiable quantum circuits (arXiv 1912.10877), behind the reference's register / block
API.  Compute runs only in ``libqbg.so`` (CUDA, built in-tree); this package is the host
mirror of the reference interface (qblock register.hpp / gates.hpp and SPEC.md blocks /
autodiff) over its C-ABI (include/qbg.h)."""
from . import errors
from ._capi import LIB_PATH, lib
from .ad import GradResult, backward, eigenbasis, expect, expect_grad, faithful_grad, obs_apply, sampled_expect
from .blocks import (CNOT, CZ, SWAP, Add, Block, Chain, Control, Daggered, GeneralMatrix, H, I2, Kron, P0, P1,
                     Pd, Phase, Program, Pu, Put, Repeat, Rotation, Rx, Ry, Rz, S, Scale, Sdag, Shift, T, Tdag,
                     Toffoli, X, Y, Z, apply, chain, compile_block, compile_observable, control, dagger,
                     define_const_gate, dispatch, gatecount, kron, mat, matblock, nparameters, parameters,
                     pauli_terms, phase, put, repeat, rot, shift, time_evolve, cache, evolve, TimeEvolution,
                     Cached, SparseOperator, sparse_operator, apply_hamiltonian, Subroutine, subroutine, is_circuit)
from .circuits import heisenberg, qft, variational_circuit
from .mmd import MMD, RBFKernel, brbf_kernel, mmd_cross, mmd_expect, mmd_grad, mmd_seed
from .register import (Register, Rng, instruct, measure, measure_collapse, probabilities, product_state, qubit_cap,
                       rand_state, set_qubit_cap, state_alloc_counter, to_text, zero_state)


def set_fusion(enabled: bool) -> None:
    """Tiled multi-gate passes (default) or one kernel per gate."""
    lib().qbg_set_fusion(1 if enabled else 0)


def set_checkpointing(enabled: bool) -> None:
    """expect' design: checkpointed (default; the forward passes keep the state after every reverse
    segment, the reverse passes read it — used when the checkpoints fit in device memory) or
    uncompute (the reverse passes uncompute ψ alongside φ̄)."""
    lib().qbg_set_checkpointing(1 if enabled else 0)


def set_checkpoint_limit(nbytes: int) -> None:
    """Upper bound on the device memory expect's checkpoints may take (-1: free memory less a
    reserve); above it the uncompute design runs."""
    lib().qbg_set_checkpoint_limit(int(nbytes))


DENSE_PATHS = {"cuda": 0, "fp64-tensor": 1, "tf32-tensor": 2}


def set_dense_path(path: str) -> None:
    """Kernel for dense 3..5-qubit gates: "fp64-tensor" (default; DMMA, complex64 widened to FP64),
    "tf32-tensor" (complex64 on tcgen05 kind::tf32, 3-piece split) or "cuda" (CUDA cores)."""
    from ._capi import check
    check(lib().qbg_set_dense_path(DENSE_PATHS[path]))


def synchronize() -> None:
    from ._capi import check
    check(lib().qbg_synchronize())
