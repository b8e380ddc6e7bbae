"""CPU: the C-ABI library loads, exports every symbol include/tfla/tfla.h
declares, and reproduces the reference's host-side validation (no compute:
there is no GPU here)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2503_14376_b200 import (BlockConfig, Dims, GeometryError, ParameterError, SequenceInputs, Variant,
                                   _ffi, chunkwise_forward)

HEADER = Path(__file__).resolve().parents[1] / "include" / "tfla" / "tfla.h"


def test_library_exports_every_header_symbol():
    declared = set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(tfla_\w+)\(", HEADER.read_text(), re.M))
    assert declared, "no declarations parsed"
    handle = _ffi.lib()
    missing = [s for s in declared if not hasattr(handle, s)]
    assert not missing, missing
    assert not _ffi.missing_symbols()
    assert set(_ffi.exported_symbols()) >= declared


def test_version_string():
    assert b"sm_100a" in _ffi.lib().tfla_version()


def _rc(d):
    return _ffi.lib().tfla_validate_dims(ctypes.byref(d._c()))


def test_dims_validation_matches_reference():
    assert _rc(Dims(T=256, L=64, d_qk=64, d_hv=64, n_head=2)) == 0
    # Dims::validate_chunked (core.cpp:9-21)
    assert _rc(Dims(T=100, L=64, d_qk=64, d_hv=64)) == _ffi.TFLA_ERR_GEOMETRY
    assert "T not divisible by L" in _ffi.last_error()
    assert _rc(Dims(T=0, L=64, d_qk=64, d_hv=64)) == _ffi.TFLA_ERR_GEOMETRY
    # kernel constraints are reported as geometry errors, never a fallback
    assert _rc(Dims(T=128, L=32, d_qk=64, d_hv=64)) == _ffi.TFLA_ERR_GEOMETRY
    assert _rc(Dims(T=128, L=64, d_qk=48, d_hv=64)) == _ffi.TFLA_ERR_GEOMETRY
    with pytest.raises(GeometryError):
        Dims(T=100, L=16, d_qk=64, d_hv=64).validate_chunked()


def test_block_validation_matches_reference():
    """test_tiled.cpp:28-40."""
    d = Dims(T=64, L=16, d_qk=16, d_hv=32)
    BlockConfig(16, 16, 16, 32).validate(d)
    BlockConfig(8, 4, 8, 16).validate(d)
    for bad in ((4, 8, 8, 16), (8, 3, 8, 16), (8, 4, 5, 16), (8, 4, 8, 12), (0, 0, 8, 16)):
        with pytest.raises(GeometryError):
            BlockConfig(*bad).validate(d)
    BlockConfig.pick_default(d).validate(d)


def test_pick_default_matches_reference():
    """BlockConfig::pick_default (tiled.cpp:32-39): caps 32/8/16/32."""
    b = BlockConfig.pick_default(Dims(T=8192, L=128, d_qk=256, d_hv=512))
    assert (b.b_lhq, b.b_lkv, b.b_dqk, b.b_dhv) == (32, 8, 16, 32)
    b = BlockConfig.pick_default(Dims(T=64, L=12, d_qk=24, d_hv=20))
    assert (b.b_lhq, b.b_lkv, b.b_dqk, b.b_dhv) == (12, 6, 12, 20)


def test_workspace_sizes():
    lib = _ffi.lib()
    d = Dims(T=8192, L=128, d_qk=256, d_hv=512, n_head=8, n_batch=8)
    f = lib.tfla_workspace_bytes(ctypes.byref(d._c()), 0, 0)
    b = lib.tfla_workspace_bytes(ctypes.byref(d._c()), 0, 1)
    s = lib.tfla_saved_state_bytes(ctypes.byref(d._c()))
    assert s == 64 * 64 * 256 * 512 * 2
    assert 0 < f < b
    assert lib.tfla_workspace_bytes(ctypes.byref(Dims(T=100, L=64, d_qk=64, d_hv=64)._c()), 0, 0) == 0


def test_null_arguments_are_parameter_errors():
    lib = _ffi.lib()
    d = Dims(T=256, L=64, d_qk=64, d_hv=64)._c()
    rc = lib.tfla_chunkwise_forward(ctypes.byref(d), 0, None, None, None, 0, None)
    assert rc == _ffi.TFLA_ERR_PARAMETER
    rc = lib.tfla_chunkwise_backward(ctypes.byref(d), 0, None, None, None, None, 0, None)
    assert rc == _ffi.TFLA_ERR_PARAMETER
    bad = Dims(T=100, L=64, d_qk=64, d_hv=64)._c()
    rc = lib.tfla_chunkwise_forward(ctypes.byref(bad), 0, None, None, None, 0, None)
    assert rc == _ffi.TFLA_ERR_GEOMETRY


def test_python_mirror_shape_errors():
    import torch

    d = Dims(T=128, L=64, d_qk=64, d_hv=64)
    z = torch.zeros
    inp = SequenceInputs(z(1, 1, 128, 64), z(1, 1, 128, 64), z(1, 1, 128, 32), z(1, 1, 128), z(1, 1, 128))
    with pytest.raises(GeometryError):
        chunkwise_forward(inp, d, Variant.Exp)
    inp.v = z(1, 1, 128, 64)
    with pytest.raises(ParameterError):  # fp32 / CPU tensors are rejected, never computed on CPU
        chunkwise_forward(inp, d, Variant.Exp)


def test_recurrent_and_init_entry_points_validate():
    """tfla_recurrent_step / tfla_chunkwise_forward_init reject bad geometry and
    missing tensors before touching the device (reference exception mapping)."""
    lib = _ffi.lib()
    dummy = ctypes.c_void_p(16)
    inp = _ffi.tfla_inputs(dummy, dummy, dummy, dummy, dummy)
    ok = Dims(T=4, L=1, d_qk=128, d_hv=256)._c()
    bad_qk = Dims(T=4, L=1, d_qk=96, d_hv=256)._c()
    bad_t = Dims(T=0, L=1, d_qk=128, d_hv=256)._c()
    assert lib.tfla_recurrent_step(ctypes.byref(bad_qk), 0, ctypes.byref(inp), dummy, dummy, dummy, dummy,
                                   None) == _ffi.TFLA_ERR_GEOMETRY
    assert lib.tfla_recurrent_step(ctypes.byref(bad_t), 0, ctypes.byref(inp), dummy, dummy, dummy, dummy,
                                   None) == _ffi.TFLA_ERR_GEOMETRY
    # mLSTMexp needs the n / m state; an unknown variant is a parameter error
    assert lib.tfla_recurrent_step(ctypes.byref(ok), 0, ctypes.byref(inp), dummy, None, None, dummy,
                                   None) == _ffi.TFLA_ERR_PARAMETER
    assert lib.tfla_recurrent_step(ctypes.byref(ok), 7, ctypes.byref(inp), dummy, dummy, dummy, dummy,
                                   None) == _ffi.TFLA_ERR_PARAMETER
    d = Dims(T=256, L=64, d_qk=64, d_hv=64)._c()
    init = _ffi.tfla_state_in(dummy, None, None)  # exp without n / m
    out = _ffi.tfla_fwd_out(dummy, None, None, dummy, dummy, dummy, None, None, None, None)
    rc = lib.tfla_chunkwise_forward_init(ctypes.byref(d), 0, ctypes.byref(inp), ctypes.byref(init), ctypes.byref(out),
                                         dummy, 1 << 40, None)
    assert rc == _ffi.TFLA_ERR_PARAMETER and "initial state" in _ffi.last_error()


def test_split_backward_entry_points_validate():
    """tfla_backward_dq / _dk / _dv need a block config (tiled.hpp:72-84), the
    saved tensors (tiled.cpp:384-386) and their outputs; the state pass and the
    assembly check their tensors -- all before any device work."""
    lib = _ffi.lib()
    dummy = ctypes.c_void_p(16)
    d = Dims(T=256, L=64, d_qk=64, d_hv=64)._c()
    blk = BlockConfig(32, 8, 16, 32)._c()
    inp = _ffi.tfla_inputs(dummy, dummy, dummy, dummy, dummy)
    sv = _ffi.tfla_bwd_in(dummy, dummy, None, dummy, dummy, dummy)
    r = ctypes.byref
    big = 1 << 40
    assert lib.tfla_backward_dq(r(d), None, 0, r(inp), r(sv), dummy, dummy, dummy, big, None) == _ffi.TFLA_ERR_PARAMETER
    assert "blocks" in _ffi.last_error()
    assert lib.tfla_backward_dq(r(d), r(blk), 0, r(inp), r(sv), dummy, None, dummy, big, None) == _ffi.TFLA_ERR_PARAMETER
    assert lib.tfla_backward_dk(r(d), r(blk), 0, r(inp), r(sv), dummy, dummy, None, dummy, dummy, big,
                                None) == _ffi.TFLA_ERR_PARAMETER
    assert lib.tfla_backward_dv(r(d), r(blk), 0, r(inp), r(sv), None, dummy, big, None) == _ffi.TFLA_ERR_PARAMETER
    nosave = _ffi.tfla_bwd_in(dummy, None, None, dummy, dummy, dummy)
    assert lib.tfla_backward_dv(r(d), r(blk), 0, r(inp), r(nosave), dummy, dummy, big, None) == _ffi.TFLA_ERR_PARAMETER
    assert "saved" in _ffi.last_error()
    bad_blk = BlockConfig(8, 32, 16, 32)._c()  # B_Lhq < B_Lkv (tiled.cpp:21-30)
    assert lib.tfla_backward_dk(r(d), r(bad_blk), 0, r(inp), r(sv), dummy, dummy, dummy, dummy, dummy, big,
                                None) == _ffi.TFLA_ERR_GEOMETRY
    assert lib.tfla_backward_state_pass(r(d), 0, r(inp), r(sv), None, None, dummy, big, None) == _ffi.TFLA_ERR_PARAMETER
    assert lib.tfla_assemble_gate_grads(r(d), 0, dummy, dummy, dummy, None, dummy, dummy, dummy, dummy,
                                        None) == _ffi.TFLA_ERR_PARAMETER
    bad = Dims(T=100, L=64, d_qk=64, d_hv=64)._c()
    assert lib.tfla_assemble_gate_grads(r(bad), 0, *([dummy] * 8), None) == _ffi.TFLA_ERR_GEOMETRY


def test_split_forward_entry_points_validate():
    """tfla_state_recurrence needs m_states and C (fp32 or bf16 copy);
    tfla_forward_parallel needs blocks and the states (n, m for mLSTMexp)."""
    lib = _ffi.lib()
    dummy = ctypes.c_void_p(16)
    r = ctypes.byref
    big = 1 << 40
    d = Dims(T=256, L=64, d_qk=64, d_hv=64)._c()
    blk = BlockConfig(32, 8, 16, 32)._c()
    inp = _ffi.tfla_inputs(dummy, dummy, dummy, dummy, dummy)
    no_c = _ffi.tfla_fwd_out(None, None, dummy, dummy, None, None, None, None, None, None)
    assert lib.tfla_state_recurrence(r(d), 0, r(inp), r(no_c), dummy, big, None) == _ffi.TFLA_ERR_PARAMETER
    no_m = _ffi.tfla_fwd_out(None, dummy, dummy, None, None, None, None, None, None, None)
    assert lib.tfla_state_recurrence(r(d), 0, r(inp), r(no_m), dummy, big, None) == _ffi.TFLA_ERR_PARAMETER
    sin = _ffi.tfla_states_in(dummy, None, dummy, dummy)
    assert lib.tfla_forward_parallel(r(d), None, 0, r(inp), r(sin), dummy, dummy, dummy, dummy, big,
                                     None) == _ffi.TFLA_ERR_PARAMETER
    sig_only_c = _ffi.tfla_states_in(None, dummy, None, None)  # fine for sig, not for exp
    assert lib.tfla_forward_parallel(r(d), r(blk), 0, r(inp), r(sig_only_c), dummy, dummy, dummy, dummy, big,
                                     None) == _ffi.TFLA_ERR_PARAMETER
    assert lib.tfla_forward_parallel(r(d), r(blk), 1, r(inp), r(sin), None, dummy, dummy, dummy, big,
                                     None) == _ffi.TFLA_ERR_PARAMETER
    bad = Dims(T=100, L=64, d_qk=64, d_hv=64)._c()
    assert lib.tfla_state_recurrence(r(bad), 0, r(inp), r(no_c), dummy, big, None) == _ffi.TFLA_ERR_GEOMETRY


def test_misaligned_device_pointers_are_parameter_errors():
    """TMA needs 16-byte aligned global addresses: a misaligned tensor is
    rejected before any device work (never a launch failure or a fault)."""
    lib = _ffi.lib()
    ok, bad = ctypes.c_void_p(1 << 20), ctypes.c_void_p((1 << 20) + 2)
    r = ctypes.byref
    d = Dims(T=256, L=64, d_qk=64, d_hv=64)._c()
    inp = _ffi.tfla_inputs(bad, ok, ok, ok, ok)
    out = _ffi.tfla_fwd_out(ok, None, None, ok, ok, ok, None, None, None, None)
    assert lib.tfla_chunkwise_forward(r(d), 0, r(inp), r(out), ok, 1 << 40, None) == _ffi.TFLA_ERR_PARAMETER
    assert "aligned" in _ffi.last_error()
    inp = _ffi.tfla_inputs(ok, ok, ok, ok, ok)
    sv = _ffi.tfla_bwd_in(bad, ok, None, ok, ok, ok)
    gr = _ffi.tfla_grads(ok, ok, ok, ok, ok)
    assert lib.tfla_chunkwise_backward(r(d), 0, r(inp), r(sv), r(gr), ok, 1 << 40, None) == _ffi.TFLA_ERR_PARAMETER
    assert "aligned" in _ffi.last_error()
    assert lib.tfla_output_norm_gate(r(d), bad, ok, ok, ctypes.c_float(1e-6), ok, None) == _ffi.TFLA_ERR_PARAMETER


def test_check_finite_validates_arguments():
    lib = _ffi.lib()
    dummy = ctypes.c_void_p(1 << 20)
    d = Dims(T=256, L=64, d_qk=64, d_hv=64)._c()
    assert lib.tfla_check_finite(ctypes.byref(d), None, None) == _ffi.TFLA_ERR_PARAMETER
    bad = _ffi.tfla_inputs(ctypes.c_void_p((1 << 20) + 2), dummy, dummy, dummy, dummy)
    assert lib.tfla_check_finite(ctypes.byref(d), ctypes.byref(bad), None) == _ffi.TFLA_ERR_PARAMETER
    assert "aligned" in _ffi.last_error()


def test_slice_count_limit():
    lib = _ffi.lib()
    d = Dims(T=64, L=64, d_qk=64, d_hv=64, n_head=256, n_batch=257)._c()
    assert lib.tfla_validate_dims(ctypes.byref(d)) == _ffi.TFLA_ERR_GEOMETRY
    assert "65535" in _ffi.last_error()


def test_kv_loop_bound_and_mask_known_answers():
    """detail::kv_block_count / block_needs_mask (tiled.cpp:43-49) through the
    C ABI, with the reference's known answers (test_tiled.cpp:42-58)."""
    from paper_2503_14376_b200 import block_needs_mask, kv_block_count

    b = BlockConfig(8, 4, 8, 16)
    assert kv_block_count(0, b) == 2
    assert kv_block_count(1, b) == 4
    assert block_needs_mask(1, 0, b)
    assert block_needs_mask(2, 0, b)
    assert not block_needs_mask(1, 1, b)
    assert block_needs_mask(2, 1, b)  # literal bound: touches the q-block start
    assert all(c <= r for r in range(8, 16) for c in range(4, 8))  # ... so the mask is a no-op there
    assert block_needs_mask(3, 1, b)
    # the bound covers every causal column of the query block (Alg. 1)
    for cfg in ((16, 16, 16, 32), (8, 4, 8, 16), (32, 8, 16, 32)):
        bc = BlockConfig(*cfg)
        for i in range(4):
            n = kv_block_count(i, bc)
            assert n * bc.b_lkv == (i + 1) * bc.b_lhq
            # blocks strictly below the query block's first row never need the mask
            for kv in range(1, n + 1):
                below = kv * bc.b_lkv < i * bc.b_lhq
                assert block_needs_mask(kv, i, bc) == (not below)
    with pytest.raises(ParameterError):
        kv_block_count(0, BlockConfig(8, 0, 8, 16))
