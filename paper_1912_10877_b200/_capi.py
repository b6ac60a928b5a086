"""ctypes binding of ``include/qbg.h`` (the C-ABI boundary).

The shared library ``libqbg.so`` is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_1912_10877_b200``).  There is no CPU fallback: if the library is missing this module
raises at import, and every device call fails with :class:`CudaError` when no GPU is present.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_uint64, c_void_p

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqbg.so")

QBG_C128, QBG_C64 = 0, 1
MAT_IDENTITY, MAT_DIAGONAL, MAT_PERMUTATION, MAT_DENSE = 0, 1, 2, 4
GEN_NONE, GEN_ROTATION, GEN_SHIFT, GEN_PHASE = 0, 1, 2, 3
MAX_TARGETS, MAX_CTRLS = 5, 16


class QbgOp(ctypes.Structure):
    _fields_ = [
        ("kind", c_int32), ("gen", c_int32), ("param", c_int32), ("ntarget", c_int32),
        ("nctrl", c_int32), ("dim", c_int32), ("targets", c_int32 * MAX_TARGETS),
        ("ctrls", c_int32 * MAX_CTRLS), ("ctrl_cfg", c_int32 * MAX_CTRLS),
        ("data", c_int64), ("perm", c_int64),
    ]


class QbgPauliTerm(ctypes.Structure):
    _fields_ = [("coef_re", c_double), ("coef_im", c_double), ("xmask", c_uint64), ("zmask", c_uint64)]


class QbgMatrix(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("dim", c_int32), ("vals", POINTER(c_double)), ("perm", POINTER(c_int64))]


assert ctypes.sizeof(QbgOp) == 192 and ctypes.sizeof(QbgPauliTerm) == 32

_ERR = {
    1: errors.ValidationError, 2: errors.ShapeError, 3: errors.RangeError, 4: errors.DispatchError,
    5: errors.ResourceError, 6: errors.UnsupportedError, 7: errors.UndecidableError,
    8: errors.RenormalizationError, 9: errors.SerializationError, 10: errors.ParseError,
    100: errors.CudaError, 101: errors.NcclError,
}

_lib = None


def lib() -> ctypes.CDLL:
    """Loads libqbg.so (once).  Fails loudly when the CUDA extension has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA engine is not built (run __graft_entry__.build()); "
            "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P = c_void_p
    sigs = {
        "qbg_last_error": (c_char_p, []), "qbg_version": (c_char_p, []),
        "qbg_set_qubit_cap": (c_int32, [c_int32]), "qbg_get_qubit_cap": (c_int32, []),
        "qbg_alloc_count": (c_uint64, []), "qbg_set_device": (c_int32, [c_int32]),
        "qbg_release_workspace": (c_int32, []),
        "qbg_load_memory": (c_int32, [P, c_int64, c_uint64, c_int32, POINTER(P)]),
        "qbg_shard_pack": (c_int32, [P, P, c_int32, c_uint64, c_int64, c_int64, P]),
        "qbg_shard_unpack": (c_int32, [P, P, c_int32, c_uint64, c_int64, c_int64, P]),
        "qbg_buffer_alloc": (c_int32, [c_int64, POINTER(P)]), "qbg_buffer_free": (c_int32, [P]),
        "qbg_set_stream": (c_int32, [P]), "qbg_synchronize": (c_int32, []),
        "qbg_set_fusion": (c_int32, [c_int32]), "qbg_set_checkpointing": (c_int32, [c_int32]), "qbg_set_checkpoint_limit": (c_int32, [c_int64]), "qbg_set_dense_path": (c_int32, [c_int32]), "qbg_profile_enable": (c_int32, [c_int32]),
        "qbg_profile_reset": (c_int32, []), "qbg_profile_report": (c_int32, [c_char_p, c_int64]),
        "qbg_launch_count": (c_uint64, []), "qbg_launch_count_reset": (c_int32, []),
        "qbg_rng_create": (c_int32, [c_uint64, POINTER(P)]), "qbg_rng_destroy": (c_int32, [P]),
        "qbg_rng_split_label": (c_int32, [P, c_char_p, POINTER(P)]),
        "qbg_rng_split_salt": (c_int32, [P, c_uint64, POINTER(P)]),
        "qbg_rng_uniform": (c_double, [P]), "qbg_rng_uniform_range": (c_double, [P, c_double, c_double]),
        "qbg_rng_gauss": (c_double, [P]), "qbg_rng_bits": (c_uint64, [P]),
        "qbg_reg_create": (c_int32, [c_int32, c_int64, c_int32, c_uint64, POINTER(P)]),
        "qbg_reg_destroy": (c_int32, [P]), "qbg_reg_clone": (c_int32, [P, POINTER(P)]),
        "qbg_reg_copy": (c_int32, [P, P]),
        "qbg_reg_info": (c_int32, [P, POINTER(c_int32), POINTER(c_int32), POINTER(c_int64), POINTER(c_int32)]),
        "qbg_reg_device_ptr": (P, [P]), "qbg_reg_rng": (P, [P]),
        "qbg_set_zero": (c_int32, [P]), "qbg_set_product": (c_int32, [P, POINTER(c_uint64), c_int64]),
        "qbg_set_rand": (c_int32, [P, c_uint64]),
        "qbg_upload": (c_int32, [P, P, c_int64]), "qbg_download": (c_int32, [P, P, c_int64]),
        "qbg_upload_raw": (c_int32, [P, P, c_int64]), "qbg_download_raw": (c_int32, [P, P, c_int64]),
        "qbg_instruct": (c_int32, [P, POINTER(QbgMatrix), POINTER(c_int32), c_int32, POINTER(c_int32),
                                   POINTER(c_int32), c_int32]),
        "qbg_instruct_tag": (c_int32, [P, c_char_p, POINTER(c_int32), c_int32, POINTER(c_int32),
                                       POINTER(c_int32), c_int32, POINTER(c_double), c_int32]),
        "qbg_norm": (c_int32, [P, P]), "qbg_inner": (c_int32, [P, P, P]),
        "qbg_scale": (c_int32, [P, c_double, c_double]), "qbg_add_scaled": (c_int32, [P, P, c_double, c_double]),
        "qbg_probabilities": (c_int32, [P, c_int64, P]),
        "qbg_measure": (c_int32, [P, c_int64, P, P]), "qbg_measure_collapse": (c_int32, [P, P, P]),
        "qbg_focus": (c_int32, [P, POINTER(c_int32), c_int32]),
        "qbg_relax": (c_int32, [P, POINTER(c_int32), c_int32, c_int32]),
        "qbg_save": (c_int32, [P, c_char_p]), "qbg_load": (c_int32, [c_char_p, c_uint64, c_int32, POINTER(P)]),
        "qbg_prog_create": (c_int32, [c_int32, POINTER(QbgOp), c_int64, P, c_int64, P, c_int64, POINTER(P)]),
        "qbg_prog_destroy": (c_int32, [P]), "qbg_prog_nparams": (c_int64, [P]),
        "qbg_prog_set_params": (c_int32, [P, P, c_int64]),
        "qbg_prog_stats": (c_int32, [P, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
        "qbg_prog_plan_info": (c_int32, [P, c_char_p, c_int64]),
        "qbg_prog_plan_preview": (c_int32, [P, c_int64, c_int32, c_char_p, c_int64]),
        "qbg_jit_check": (c_int32, [P, P, c_int64, c_int32, POINTER(c_int64)]),
        "qbg_jit_stats": (c_int32, [POINTER(c_int64), POINTER(c_int64)]),
        "qbg_apply": (c_int32, [P, P]), "qbg_apply_adjoint": (c_int32, [P, P]),
        "qbg_obs_create": (c_int32, [c_int32, POINTER(QbgPauliTerm), c_int64, POINTER(P)]),
        "qbg_obs_destroy": (c_int32, [P]), "qbg_expect": (c_int32, [P, P, P]),
        "qbg_obs_apply": (c_int32, [P, P, P]), "qbg_backward": (c_int32, [P, P, P, P]),
        "qbg_expect_grad": (c_int32, [P, P, P, c_int32, P, P, P]),
        "qbg_mmd_create": (c_int32, [c_int32, P, P, c_int32, POINTER(P)]), "qbg_mmd_destroy": (c_int32, [P]),
        "qbg_mmd_band": (c_int32, [P, POINTER(c_int32)]), "qbg_mmd_loss": (c_int32, [P, P, P]),
        "qbg_mmd_seed": (c_int32, [P, P, P, P]), "qbg_mmd_cross": (c_int32, [P, P, P, P]),
        "qbg_mmd_grad": (c_int32, [P, P, P, c_int32, P, P, P]),
        "qbg_time_evolve": (c_int32, [P, P, c_double, c_double, c_int32, POINTER(c_int32)]),
        "qbg_run_program": (c_int32, [P, P, c_int64, P, c_int64, P, c_int64, P, c_int64]),
        "qbg_expect_pauli_sum": (c_int32, [P, POINTER(QbgPauliTerm), c_int64, P]),
        "qbg_axpy": (c_int32, [P, P, c_double, c_double]), "qbg_collapse": (c_int32, [P, P, P]),
        "qbg_sparse_create": (c_int32, [c_int32, c_int64, P, P, P, POINTER(P)]),
        "qbg_sparse_destroy": (c_int32, [P]), "qbg_sparse_apply": (c_int32, [P, P, P]),
        "qbg_time_evolve_sparse": (c_int32, [P, P, c_double, c_double, c_int32, POINTER(c_int32)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = None  # filled lazily by exported_symbols()


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().qbg_last_error().decode(errors="replace")
        raise _ERR.get(rc, errors.Error)(msg)


def i32(seq):
    seq = list(seq)
    return (c_int32 * max(1, len(seq)))(*seq), len(seq)
