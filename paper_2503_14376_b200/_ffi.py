"""ctypes binding of the C ABI in ``include/tfla/tfla.h`` (libtfla_b200.so).

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``)
into ``paper_2503_14376_b200/_lib``. Importing this module never falls back to
anything: if the library is missing, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libtfla_b200.so"

TFLA_OK = 0
TFLA_ERR_GEOMETRY = 1
TFLA_ERR_PARAMETER = 2
TFLA_ERR_NUMERIC = 3
TFLA_ERR_CUDA = 4

VARIANT_EXP = 0
VARIANT_SIG = 1


class tfla_dims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("T", "L", "d_qk", "d_hv", "n_head", "n_batch")]


class tfla_blocks(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("b_lhq", "b_lkv", "b_dqk", "b_dhv")]


class tfla_inputs(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("q", "k", "v", "i_pre", "f_pre")]


class tfla_fwd_out(ctypes.Structure):
    _fields_ = [
        (n, ctypes.c_void_p)
        for n in (
            "h",
            "c_states",
            "n_states",
            "m_states",
            "m_combine",
            "h_denom",
            "c_final",
            "n_final",
            "m_final",
            "saved_states",
        )
    ]


class tfla_state_in(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("c", "n", "m")]


class tfla_bwd_in(ctypes.Structure):
    _fields_ = [
        (n, ctypes.c_void_p)
        for n in ("d_h", "saved_states", "c_states", "m_states", "m_combine", "h_denom")
    ]


class tfla_states_in(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("saved_states", "c_states", "n_states", "m_states")]


class tfla_grads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("dq", "dk", "dv", "d_fpre", "d_ipre")]


# name -> (restype, argtypes)
_SIGNATURES = {
    "tfla_validate_dims": (ctypes.c_int, [ctypes.POINTER(tfla_dims)]),
    "tfla_validate_blocks": (ctypes.c_int, [ctypes.POINTER(tfla_dims), ctypes.POINTER(tfla_blocks)]),
    "tfla_pick_default_blocks": (ctypes.c_int, [ctypes.POINTER(tfla_dims), ctypes.POINTER(tfla_blocks)]),
    "tfla_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(tfla_dims), ctypes.c_int, ctypes.c_int]),
    "tfla_saved_state_bytes": (ctypes.c_size_t, [ctypes.POINTER(tfla_dims)]),
    "tfla_chunkwise_forward": (
        ctypes.c_int,
        [
            ctypes.POINTER(tfla_dims),
            ctypes.c_int,
            ctypes.POINTER(tfla_inputs),
            ctypes.POINTER(tfla_fwd_out),
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "tfla_forward": (
        ctypes.c_int,
        [
            ctypes.POINTER(tfla_dims),
            ctypes.POINTER(tfla_blocks),
            ctypes.c_int,
            ctypes.POINTER(tfla_inputs),
            ctypes.POINTER(tfla_fwd_out),
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "tfla_chunkwise_backward": (
        ctypes.c_int,
        [
            ctypes.POINTER(tfla_dims),
            ctypes.c_int,
            ctypes.POINTER(tfla_inputs),
            ctypes.POINTER(tfla_bwd_in),
            ctypes.POINTER(tfla_grads),
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "tfla_backward": (
        ctypes.c_int,
        [
            ctypes.POINTER(tfla_dims),
            ctypes.POINTER(tfla_blocks),
            ctypes.c_int,
            ctypes.POINTER(tfla_inputs),
            ctypes.POINTER(tfla_bwd_in),
            ctypes.POINTER(tfla_grads),
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "tfla_chunkwise_forward_init": (
        ctypes.c_int,
        [
            ctypes.POINTER(tfla_dims),
            ctypes.c_int,
            ctypes.POINTER(tfla_inputs),
            ctypes.POINTER(tfla_state_in),
            ctypes.POINTER(tfla_fwd_out),
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "tfla_chunkwise_gates": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_int] + [ctypes.c_void_p] * 5 + [ctypes.c_void_p],
    ),
    "tfla_train_step_host": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_int, ctypes.POINTER(tfla_inputs), ctypes.c_void_p,
         ctypes.POINTER(tfla_grads), ctypes.c_void_p, ctypes.c_void_p],
    ),
    "tfla_check_finite": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.POINTER(tfla_inputs), ctypes.c_void_p],
    ),
    "tfla_state_recurrence": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_int, ctypes.POINTER(tfla_inputs), ctypes.POINTER(tfla_fwd_out),
         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "tfla_forward_parallel": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.POINTER(tfla_blocks), ctypes.c_int, ctypes.POINTER(tfla_inputs),
         ctypes.POINTER(tfla_states_in), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_size_t, ctypes.c_void_p],
    ),
    "tfla_backward_dq": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.POINTER(tfla_blocks), ctypes.c_int, ctypes.POINTER(tfla_inputs),
         ctypes.POINTER(tfla_bwd_in), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
         ctypes.c_void_p],
    ),
    "tfla_backward_dk": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.POINTER(tfla_blocks), ctypes.c_int, ctypes.POINTER(tfla_inputs),
         ctypes.POINTER(tfla_bwd_in), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "tfla_backward_dv": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.POINTER(tfla_blocks), ctypes.c_int, ctypes.POINTER(tfla_inputs),
         ctypes.POINTER(tfla_bwd_in), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "tfla_backward_state_pass": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_int, ctypes.POINTER(tfla_inputs), ctypes.POINTER(tfla_bwd_in),
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "tfla_assemble_gate_grads": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_int] + [ctypes.c_void_p] * 8 + [ctypes.c_void_p],
    ),
    "tfla_apply_gate_softcap": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p],
    ),
    "tfla_chunkwise_forward_f32": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_int, ctypes.POINTER(tfla_inputs), ctypes.POINTER(tfla_fwd_out),
         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "tfla_chunkwise_forward_gated": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_int, ctypes.POINTER(tfla_inputs), ctypes.POINTER(tfla_fwd_out),
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
         ctypes.c_void_p],
    ),
    "tfla_output_norm_gate": (
        ctypes.c_int,
        [ctypes.POINTER(tfla_dims), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float,
         ctypes.c_void_p, ctypes.c_void_p],
    ),
    "tfla_recurrent_step": (
        ctypes.c_int,
        [
            ctypes.POINTER(tfla_dims),
            ctypes.c_int,
            ctypes.POINTER(tfla_inputs),
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
        ],
    ),
    "tfla_kv_block_count": (ctypes.c_int64, [ctypes.c_int64, ctypes.POINTER(tfla_blocks)]),
    "tfla_block_needs_mask": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(tfla_blocks)]),
    "tfla_chunkwise_forward_frozen": (
        ctypes.c_int,
        [
            ctypes.POINTER(tfla_dims),
            ctypes.c_int,
            ctypes.POINTER(tfla_inputs),
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "tfla_stab_enable": (ctypes.c_int, [ctypes.c_int]),
    "tfla_stab_read": (
        ctypes.c_int,
        [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)],
    ),
    "tfla_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "tfla_profile_read": (
        ctypes.c_int,
        [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), ctypes.c_int],
    ),
    "tfla_profile_name": (ctypes.c_char_p, [ctypes.c_int]),
    "tfla_last_error": (ctypes.c_char_p, []),
    "tfla_version": (ctypes.c_char_p, []),
    "tfla_selftest_gemm": (
        ctypes.c_int,
        [
            ctypes.c_int,
            ctypes.c_int,
            ctypes.c_int,
            ctypes.c_int,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
        ],
    ),
}

_lib = None


def lib_path() -> Path:
    return Path(os.environ.get("TFLA_B200_LIB", _LIB_PATH))


def lib() -> ctypes.CDLL:
    """Load libtfla_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not path.exists():
            raise RuntimeError(
                f"libtfla_b200.so not built at {path}; run `make` or __graft_entry__.build()"
            )
        handle = ctypes.CDLL(str(path))
        for name, (res, args) in _SIGNATURES.items():
            try:
                fn = getattr(handle, name)
            except AttributeError:  # reported by missing_symbols() / the export test
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def missing_symbols() -> list[str]:
    handle = lib()
    out = []
    for name in _SIGNATURES:
        try:
            getattr(handle, name)
        except AttributeError:
            out.append(name)
    return out


def last_error() -> str:
    msg = lib().tfla_last_error()
    return msg.decode() if msg else ""
