"""Python mirror of the reference ``mlstm::`` API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/mlstm/{core,chunkwise,tiled}.hpp), on device
tensors: q/k/v in bf16, gates / states / stats in fp32. Every call goes
through ``libtfla_b200.so`` (hand-written sm_100a kernels); there is no CPU or
PyTorch fallback -- a missing library or device raises.

    Reference                              Here
    mlstm::Dims (core.hpp:27-39)           Dims
    mlstm::BlockConfig (tiled.hpp:12-22)   BlockConfig
    mlstm::Variant (core.hpp:113)          Variant
    SequenceInputs (core.hpp:147-153)      SequenceInputs (torch tensors)
    ChunkwiseForward (chunkwise.hpp:25-29) ChunkwiseForward
    Gradients (chunkwise.hpp:32-35)        Gradients
    chunkwise_forward / tfla_forward       same names
    chunkwise_backward / tfla_backward     same names
    GeometryError / ParameterError / NumericError (core.hpp:11-23)  same names
"""
from __future__ import annotations

import ctypes
import enum
import functools
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _ffi


class GeometryError(ValueError):
    """mlstm::GeometryError: inconsistent shapes or chunk geometry."""


class ParameterError(ValueError):
    """mlstm::ParameterError: out-of-range parameters / missing saved tensors."""


class NumericError(RuntimeError):
    """mlstm::NumericError: non-finite inputs."""


class CudaError(RuntimeError):
    """Launch or driver failure inside libtfla_b200."""


_ERRORS = {
    _ffi.TFLA_ERR_GEOMETRY: GeometryError,
    _ffi.TFLA_ERR_PARAMETER: ParameterError,
    _ffi.TFLA_ERR_NUMERIC: NumericError,
    _ffi.TFLA_ERR_CUDA: CudaError,
}


def _check(rc: int) -> None:
    if rc != _ffi.TFLA_OK:
        raise _ERRORS.get(rc, CudaError)(_ffi.last_error())


def _tensor_device(obj):
    if isinstance(obj, torch.Tensor):
        return obj.device if obj.is_cuda else None
    for name in ("q", "h_tilde", "C"):  # SequenceInputs / MemoryState
        t = getattr(obj, name, None)
        if isinstance(t, torch.Tensor) and t.is_cuda:
            return t.device
    return None


def _on_input_device(fn):
    """Run ``fn`` with the inputs' CUDA device current: the C ABI launches on
    the current device and its stream, and the workspace cache is keyed by that
    device's stream, so a call on cuda:N with another device current would mix
    devices. Every tensor argument must live on that one device."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        devs = {d for d in (_tensor_device(a) for a in (*args, *kwargs.values())) if d is not None}
        for a in (*args, *kwargs.values()):
            if hasattr(a, "__dataclass_fields__"):
                devs |= {t.device for t in vars(a).values() if isinstance(t, torch.Tensor) and t.is_cuda}
        if len(devs) > 1:
            raise ParameterError(f"{fn.__name__}: tensors on several devices {sorted(map(str, devs))}")
        if not devs:
            return fn(*args, **kwargs)
        with torch.cuda.device(devs.pop()):
            return fn(*args, **kwargs)

    return wrapper


class Variant(enum.IntEnum):
    Exp = _ffi.VARIANT_EXP
    Sig = _ffi.VARIANT_SIG


@dataclass
class Dims:
    T: int = 1
    L: int = 1
    d_qk: int = 1
    d_hv: int = 1
    n_head: int = 1
    n_batch: int = 1

    def n_chunk(self) -> int:
        return self.T // self.L

    def _c(self) -> _ffi.tfla_dims:
        return _ffi.tfla_dims(self.T, self.L, self.d_qk, self.d_hv, self.n_head, self.n_batch)

    def validate_chunked(self) -> None:
        _check(_ffi.lib().tfla_validate_dims(ctypes.byref(self._c())))


@dataclass
class BlockConfig:
    b_lhq: int = 0
    b_lkv: int = 0
    b_dqk: int = 0
    b_dhv: int = 0

    def _c(self) -> _ffi.tfla_blocks:
        return _ffi.tfla_blocks(self.b_lhq, self.b_lkv, self.b_dqk, self.b_dhv)

    def validate(self, dims: Dims) -> None:
        _check(_ffi.lib().tfla_validate_blocks(ctypes.byref(dims._c()), ctypes.byref(self._c())))

    @staticmethod
    def pick_default(dims: Dims) -> "BlockConfig":
        out = _ffi.tfla_blocks()
        _check(_ffi.lib().tfla_pick_default_blocks(ctypes.byref(dims._c()), ctypes.byref(out)))
        return BlockConfig(out.b_lhq, out.b_lkv, out.b_dqk, out.b_dhv)


@dataclass
class SequenceInputs:
    q: torch.Tensor  # bf16 [B,H,T,dqk]
    k: torch.Tensor  # bf16 [B,H,T,dqk]
    v: torch.Tensor  # bf16 [B,H,T,dhv]
    i_pre: torch.Tensor  # fp32 [B,H,T]
    f_pre: torch.Tensor  # fp32 [B,H,T]

    def validate(self, dims: Dims, operand_dtype=None) -> None:
        """SequenceInputs::validate (core.cpp:106-117) -- shapes, dtypes, device.
        q / k / v are bf16 (the tensor-core path) or fp32 (``chunkwise_forward_f32``)."""
        od = operand_dtype or torch.bfloat16
        qk = (dims.n_batch, dims.n_head, dims.T, dims.d_qk)
        hv = (dims.n_batch, dims.n_head, dims.T, dims.d_hv)
        g = (dims.n_batch, dims.n_head, dims.T)
        if tuple(self.q.shape) != qk or tuple(self.k.shape) != qk:
            raise GeometryError("q/k shape mismatch with dims")
        if tuple(self.v.shape) != hv:
            raise GeometryError("v shape mismatch with dims")
        if tuple(self.i_pre.shape) != g or tuple(self.f_pre.shape) != g:
            raise GeometryError("gate pre-activation shape mismatch with dims")
        for name, t, dt in (("q", self.q, od), ("k", self.k, od),
                            ("v", self.v, od), ("i_pre", self.i_pre, torch.float32),
                            ("f_pre", self.f_pre, torch.float32)):
            if t.dtype != dt:
                raise ParameterError(f"{name} must be {dt}")
            if not t.is_cuda:
                raise ParameterError(f"{name} must be a CUDA tensor")
            if not t.is_contiguous():
                raise ParameterError(f"{name} must be contiguous")

    @_on_input_device
    def check_finite(self, dims: "Dims") -> None:
        """The reference's all_finite check (core.cpp:114-116), on demand, as a
        device pass of the library (tfla_check_finite -> NumericError)."""
        self.validate(dims)
        _check(_ffi.lib().tfla_check_finite(ctypes.byref(dims._c()), ctypes.byref(self._c()), _stream()))

    def _c(self) -> _ffi.tfla_inputs:
        return _ffi.tfla_inputs(self.q.data_ptr(), self.k.data_ptr(), self.v.data_ptr(),
                                self.i_pre.data_ptr(), self.f_pre.data_ptr())


@dataclass
class ChunkStates:
    C: Optional[torch.Tensor]  # fp32 [B,H,NC+1,dqk,dhv] (None when not requested)
    n: Optional[torch.Tensor]  # fp32 [B,H,NC+1,dqk]
    m: torch.Tensor  # fp32 [B,H,NC+1]


@dataclass
class SavedStats:
    m_combine: torch.Tensor  # fp32 [B,H,T]
    h_denom: torch.Tensor  # fp32 [B,H,T]


@dataclass
class ChunkwiseForward:
    h_tilde: torch.Tensor  # bf16 [B,H,T,dhv]
    states: ChunkStates
    stats: SavedStats
    saved_states: Optional[torch.Tensor] = None  # bf16 [B,H,NC,dqk,dhv]: backward operand copy
    C_final: Optional[torch.Tensor] = None  # fp32 [B,H,dqk,dhv]
    n_final: Optional[torch.Tensor] = None
    m_final: Optional[torch.Tensor] = None


@dataclass
class Gradients:
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor
    d_fpre: torch.Tensor
    d_ipre: torch.Tensor


_WS: dict = {}


def _workspace(dims: Dims, variant: Variant, pass_: int, device) -> torch.Tensor:
    nbytes = _ffi.lib().tfla_workspace_bytes(ctypes.byref(dims._c()), int(variant), pass_)
    if nbytes == 0:
        dims.validate_chunked()
        raise ParameterError("workspace size query failed")
    # one cache entry per (device, pass, stream): calls on one stream are
    # ordered, calls on different streams must not share scratch memory
    key = (str(device), pass_, torch.cuda.current_stream(device).cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _forward(inputs: SequenceInputs, dims: Dims, variant: Variant, blocks: Optional[BlockConfig],
             all_states: bool, keep_saved: bool, initial_state=None, out_gate=None):
    dims.validate_chunked()
    if blocks is not None:
        blocks.validate(dims)
    inputs.validate(dims)
    dev = inputs.q.device
    B, H, T, NC = dims.n_batch, dims.n_head, dims.T, dims.n_chunk()
    f32 = dict(dtype=torch.float32, device=dev)
    h = torch.empty(B, H, T, dims.d_hv, dtype=torch.bfloat16, device=dev)
    C = torch.empty(B, H, NC + 1, dims.d_qk, dims.d_hv, **f32) if all_states else None
    n = torch.empty(B, H, NC + 1, dims.d_qk, **f32) if all_states else None
    m = torch.empty(B, H, NC + 1, **f32)
    mc = torch.empty(B, H, T, **f32)
    hd = torch.empty(B, H, T, **f32)
    Cf = torch.empty(B, H, dims.d_qk, dims.d_hv, **f32)
    nf = torch.empty(B, H, dims.d_qk, **f32)
    mf = torch.empty(B, H, **f32)
    saved = (torch.empty(B, H, NC, dims.d_qk, dims.d_hv, dtype=torch.bfloat16, device=dev)
             if keep_saved else None)
    out = _ffi.tfla_fwd_out(
        h.data_ptr(), C.data_ptr() if C is not None else None, n.data_ptr() if n is not None else None,
        m.data_ptr(), mc.data_ptr(), hd.data_ptr(), Cf.data_ptr(), nf.data_ptr(), mf.data_ptr(),
        saved.data_ptr() if saved is not None else None)
    ws = _workspace(dims, variant, 0, dev)
    lib = _ffi.lib()
    y = None
    if out_gate is not None:
        o_pre, gamma, eps = out_gate
        if tuple(o_pre.shape) != (B, H, T, dims.d_hv):
            raise GeometryError("o_pre must be [B,H,T,dhv]")
        if tuple(gamma.shape) != (H, dims.d_hv):
            raise GeometryError("gamma must be [H, dhv]")
        for name, t, dt in (("o_pre", o_pre, torch.bfloat16), ("gamma", gamma, torch.float32)):
            if t.dtype != dt or t.device != dev or not t.is_contiguous():
                raise ParameterError(f"{name} must be a contiguous {dt} tensor on the inputs' device")
        y = torch.empty(B, H, T, dims.d_hv, dtype=torch.bfloat16, device=dev)
        rc = lib.tfla_chunkwise_forward_gated(ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()),
                                              ctypes.byref(out), o_pre.data_ptr(), gamma.data_ptr(), float(eps),
                                              y.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    elif initial_state is not None:
        if blocks is not None:
            raise ParameterError("an initial state is supported on chunkwise_forward only")
        B_, H_ = dims.n_batch, dims.n_head
        for name, t, shape in (("C", initial_state.C, (B_, H_, dims.d_qk, dims.d_hv)),
                               ("n", initial_state.n, (B_, H_, dims.d_qk)), ("m", initial_state.m, (B_, H_))):
            if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous():
                raise GeometryError(f"initial state {name} must be contiguous fp32 {shape}")
        init = _ffi.tfla_state_in(initial_state.C.data_ptr(), initial_state.n.data_ptr(),
                                  initial_state.m.data_ptr())
        rc = lib.tfla_chunkwise_forward_init(ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()),
                                             ctypes.byref(init), ctypes.byref(out), ws.data_ptr(), ws.numel(),
                                             _stream())
    elif blocks is None:
        rc = lib.tfla_chunkwise_forward(ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()),
                                        ctypes.byref(out), ws.data_ptr(), ws.numel(), _stream())
    else:
        rc = lib.tfla_forward(ctypes.byref(dims._c()), ctypes.byref(blocks._c()), int(variant),
                              ctypes.byref(inputs._c()), ctypes.byref(out), ws.data_ptr(), ws.numel(),
                              _stream())
    _check(rc)
    fwd = ChunkwiseForward(h, ChunkStates(C, n, m), SavedStats(mc, hd), saved, Cf, nf, mf)
    return fwd if out_gate is None else (fwd, y)


@_on_input_device
def chunkwise_forward(inputs: SequenceInputs, dims: Dims, variant: Variant, *,
                      all_states: bool = True, keep_saved: bool = True,
                      initial_state: Optional["MemoryState"] = None) -> ChunkwiseForward:
    """chunkwise_forward (chunkwise.hpp:39-40); ``initial_state`` continues an
    earlier segment (the chunkwise analogue of RecurrentOptions::initial_state,
    recurrent.hpp:23-27)."""
    return _forward(inputs, dims, Variant(variant), None, all_states, keep_saved, initial_state)


@_on_input_device
def chunkwise_forward_f32(inputs: SequenceInputs, dims: Dims, variant: Variant, *,
                          all_states: bool = True) -> ChunkwiseForward:
    """chunkwise_forward on fp32 operands (the reference's <float, float>
    instantiation, chunkwise.cpp:183-194; BASELINE config 0 as worded): fp32
    q / k / v, fp32 h_tilde and states (tfla_chunkwise_forward_f32, CUDA cores)."""
    dims.validate_chunked()
    inputs.validate(dims, operand_dtype=torch.float32)
    dev = inputs.q.device
    B, H, T, NC = dims.n_batch, dims.n_head, dims.T, dims.n_chunk()
    f32 = dict(dtype=torch.float32, device=dev)
    h = torch.empty(B, H, T, dims.d_hv, **f32)
    C = torch.empty(B, H, NC + 1, dims.d_qk, dims.d_hv, **f32) if all_states else None
    n = torch.empty(B, H, NC + 1, dims.d_qk, **f32) if all_states else None
    m = torch.empty(B, H, NC + 1, **f32)
    mc, hd = torch.empty(B, H, T, **f32), torch.empty(B, H, T, **f32)
    Cf, nf, mf = torch.empty(B, H, dims.d_qk, dims.d_hv, **f32), torch.empty(B, H, dims.d_qk, **f32), torch.empty(B, H, **f32)
    out = _ffi.tfla_fwd_out(h.data_ptr(), C.data_ptr() if C is not None else None,
                            n.data_ptr() if n is not None else None, m.data_ptr(), mc.data_ptr(), hd.data_ptr(),
                            Cf.data_ptr(), nf.data_ptr(), mf.data_ptr(), None)
    ws = _workspace(dims, Variant(variant), 0, dev)
    _check(_ffi.lib().tfla_chunkwise_forward_f32(ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()),
                                                 ctypes.byref(out), ws.data_ptr(), ws.numel(), _stream()))
    return ChunkwiseForward(h, ChunkStates(C, n, m), SavedStats(mc, hd), None, Cf, nf, mf)


@_on_input_device
def chunkwise_forward_gated(inputs: SequenceInputs, dims: Dims, variant: Variant, o_pre: torch.Tensor,
                            gamma: torch.Tensor, eps: float = 1e-6, *, all_states: bool = True,
                            keep_saved: bool = True):
    """chunkwise_forward with the mLSTM cell output (eq. 5) fused into the
    H store: returns (ChunkwiseForward, y) with y = sigmoid(o_pre) * rms_norm(h_tilde;
    gamma[h], eps) (transfer.cpp:8-18) -- output_norm_gate(fwd.h_tilde, o_pre, gamma,
    eps) without the second pass over h_tilde (tfla_chunkwise_forward_gated)."""
    if not eps >= 0.0:
        raise ParameterError("rms_norm: eps must be >= 0")
    return _forward(inputs, dims, Variant(variant), None, all_states, keep_saved, None, (o_pre, gamma, eps))


@_on_input_device
def chunkwise_forward_frozen(inputs: SequenceInputs, dims: Dims, variant: Variant, frozen_states: ChunkStates,
                             frozen_stats: SavedStats) -> torch.Tensor:
    """chunkwise_forward_frozen (chunkwise.hpp:42-46 / chunkwise.cpp:304-394):
    the forward with the max-state schedule, m_combine and h_denom pinned to
    saved values -- the function tfla_chunkwise_backward differentiates."""
    dims.validate_chunked()
    inputs.validate(dims)
    if frozen_states.m is None or frozen_stats.m_combine is None or frozen_stats.h_denom is None:
        raise ParameterError("chunkwise_forward_frozen: missing saved stats")
    B, H, T, NC = dims.n_batch, dims.n_head, dims.T, dims.n_chunk()
    for name, t, shape in (("m", frozen_states.m, (B, H, NC + 1)), ("m_combine", frozen_stats.m_combine, (B, H, T)),
                           ("h_denom", frozen_stats.h_denom, (B, H, T))):
        if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous():
            raise GeometryError(f"frozen {name} must be contiguous fp32 {shape}")
    h = torch.empty(B, H, T, dims.d_hv, dtype=torch.bfloat16, device=inputs.q.device)
    ws = _workspace(dims, Variant(variant), 0, inputs.q.device)
    _check(_ffi.lib().tfla_chunkwise_forward_frozen(
        ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()), frozen_states.m.data_ptr(),
        frozen_stats.m_combine.data_ptr(), frozen_stats.h_denom.data_ptr(), h.data_ptr(), ws.data_ptr(),
        ws.numel(), _stream()))
    return h


class stab:
    """mlstm::stab (core.cpp:145-166) for the device kernels: an opt-in audit
    of every stabilised exponent (tfla_stab_enable / tfla_stab_read)."""

    @staticmethod
    def enable(on: bool = True) -> None:
        _check(_ffi.lib().tfla_stab_enable(1 if on else 0))

    @staticmethod
    def read() -> tuple:
        """(checks, violations, max_arg) since the last read; resets them."""
        c, v, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        _check(_ffi.lib().tfla_stab_read(ctypes.byref(c), ctypes.byref(v), ctypes.byref(m)))
        return c.value, v.value, m.value

    @staticmethod
    def reset() -> None:
        stab.read()


def kv_block_count(i_lq: int, blocks: BlockConfig) -> int:
    """detail::kv_block_count (tiled.cpp:43-45)."""
    r = _ffi.lib().tfla_kv_block_count(int(i_lq), ctypes.byref(blocks._c()))
    if r < 0:
        raise ParameterError("kv_block_count: bad arguments")
    return r


def block_needs_mask(i_kv_1based: int, i_lq: int, blocks: BlockConfig) -> bool:
    """detail::block_needs_mask (tiled.cpp:47-49)."""
    r = _ffi.lib().tfla_block_needs_mask(int(i_kv_1based), int(i_lq), ctypes.byref(blocks._c()))
    if r < 0:
        raise ParameterError("block_needs_mask: bad arguments")
    return bool(r)


@_on_input_device
def tfla_forward(inputs: SequenceInputs, dims: Dims, blocks: BlockConfig, variant: Variant, *,
                 all_states: bool = True, keep_saved: bool = True) -> ChunkwiseForward:
    """tfla_forward (tiled.hpp:51-52)."""
    return _forward(inputs, dims, Variant(variant), blocks, all_states, keep_saved)


def _bwd_in(inputs: SequenceInputs, dims: Dims, d_h: torch.Tensor, states: ChunkStates,
            stats: SavedStats, blocks: Optional[BlockConfig], saved_states: Optional[torch.Tensor]):
    """Shared argument checks of the backward entry points (tiled.cpp:378-387)."""
    dims.validate_chunked()
    if blocks is not None:
        blocks.validate(dims)
    inputs.validate(dims)
    if states is None or stats is None or states.m is None or stats.m_combine is None \
            or stats.h_denom is None or (saved_states is None and states.C is None):
        raise ParameterError("chunkwise_backward: missing saved forward tensors")
    if tuple(d_h.shape) != tuple(inputs.v.shape):
        raise GeometryError("chunkwise_backward: dH shape mismatch")
    d_h = d_h.to(torch.bfloat16).contiguous()
    bin_ = _ffi.tfla_bwd_in(
        d_h.data_ptr(), saved_states.data_ptr() if saved_states is not None else None,
        states.C.data_ptr() if states.C is not None else None, states.m.data_ptr(),
        stats.m_combine.data_ptr(), stats.h_denom.data_ptr())
    return d_h, bin_


def _backward(inputs: SequenceInputs, dims: Dims, variant: Variant, d_h: torch.Tensor,
              states: ChunkStates, stats: SavedStats, blocks: Optional[BlockConfig],
              saved_states: Optional[torch.Tensor]) -> Gradients:
    d_h, bin_ = _bwd_in(inputs, dims, d_h, states, stats, blocks, saved_states)
    dev = inputs.q.device
    dq = torch.empty_like(inputs.q)
    dk = torch.empty_like(inputs.k)
    dv = torch.empty_like(inputs.v)
    dfp = torch.empty_like(inputs.f_pre)
    dip = torch.empty_like(inputs.i_pre)
    gr = _ffi.tfla_grads(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), dfp.data_ptr(), dip.data_ptr())
    ws = _workspace(dims, variant, 1, dev)
    lib = _ffi.lib()
    if blocks is None:
        rc = lib.tfla_chunkwise_backward(ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()),
                                         ctypes.byref(bin_), ctypes.byref(gr), ws.data_ptr(), ws.numel(),
                                         _stream())
    else:
        rc = lib.tfla_backward(ctypes.byref(dims._c()), ctypes.byref(blocks._c()), int(variant),
                               ctypes.byref(inputs._c()), ctypes.byref(bin_), ctypes.byref(gr),
                               ws.data_ptr(), ws.numel(), _stream())
    _check(rc)
    return Gradients(dq, dk, dv, dfp, dip)


@_on_input_device
def chunkwise_backward(inputs: SequenceInputs, dims: Dims, variant: Variant, d_h: torch.Tensor,
                       states: ChunkStates, stats: SavedStats,
                       saved_states: Optional[torch.Tensor] = None) -> Gradients:
    """chunkwise_backward (chunkwise.hpp:52-54)."""
    return _backward(inputs, dims, Variant(variant), d_h, states, stats, None, saved_states)


@_on_input_device
def tfla_backward(inputs: SequenceInputs, dims: Dims, blocks: BlockConfig, variant: Variant,
                  d_h: torch.Tensor, states: ChunkStates, stats: SavedStats,
                  saved_states: Optional[torch.Tensor] = None) -> Gradients:
    """tfla_backward (tiled.hpp:88-90)."""
    return _backward(inputs, dims, Variant(variant), d_h, states, stats, blocks, saved_states)


# ---------------------------------------------------------------- gates
@dataclass
class ChunkwiseGates:
    """ChunkwiseGates (gates.hpp:21-29) for every head, f64 on the device."""
    g_sum: torch.Tensor  # [B,H,NC]
    b_cum: torch.Tensor  # [B,H,T]
    a_tail: torch.Tensor  # [B,H,T]


@_on_input_device
def chunkwise_gates(f_pre: torch.Tensor, i_pre: torch.Tensor, dims: Dims, variant: Variant) -> ChunkwiseGates:
    """chunkwise_gates (gates.hpp:31-35 / gates.cpp:20-59) on the device."""
    dims.validate_chunked()
    B, H, T, NC = dims.n_batch, dims.n_head, dims.T, dims.n_chunk()
    for name, t in (("f_pre", f_pre), ("i_pre", i_pre)):
        if tuple(t.shape) != (B, H, T) or t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ParameterError(f"chunkwise_gates: {name} must be contiguous CUDA fp32 {(B, H, T)}")
    f64 = dict(dtype=torch.float64, device=f_pre.device)
    out = ChunkwiseGates(torch.empty(B, H, NC, **f64), torch.empty(B, H, T, **f64), torch.empty(B, H, T, **f64))
    _check(_ffi.lib().tfla_chunkwise_gates(ctypes.byref(dims._c()), int(variant), f_pre.data_ptr(), i_pre.data_ptr(),
                                           out.g_sum.data_ptr(), out.b_cum.data_ptr(), out.a_tail.data_ptr(),
                                           _stream()))
    return out


# ---------------------------------------------------------------- host-buffer training step
@_on_input_device
def train_step_host(inputs: SequenceInputs, dims: Dims, variant: Variant, d_h: torch.Tensor):
    """One forward + backward with HOST tensors in and out (tfla_train_step_host):
    the reference's host-tensor boundary (chunkwise.hpp:39-54) for a training
    step. ``inputs`` / ``d_h`` are CPU tensors (pin them for the PCIe rate);
    returns (h_tilde, Gradients) as CPU tensors. Stream-ordered on the current
    CUDA stream; synchronises it before returning."""
    dims.validate_chunked()
    B, H, T = dims.n_batch, dims.n_head, dims.T
    shapes = (("q", inputs.q, (B, H, T, dims.d_qk), torch.bfloat16), ("k", inputs.k, (B, H, T, dims.d_qk), torch.bfloat16),
              ("v", inputs.v, (B, H, T, dims.d_hv), torch.bfloat16), ("i_pre", inputs.i_pre, (B, H, T), torch.float32),
              ("f_pre", inputs.f_pre, (B, H, T), torch.float32), ("d_h", d_h, (B, H, T, dims.d_hv), torch.bfloat16))
    for name, t, shape, dt in shapes:
        if tuple(t.shape) != shape:
            raise GeometryError(f"train_step_host: {name} shape {tuple(t.shape)} != {shape}")
        if t.dtype != dt or t.is_cuda or not t.is_contiguous():
            raise ParameterError(f"train_step_host: {name} must be a contiguous host {dt} tensor")
    pin = inputs.q.is_pinned()
    h = torch.empty(B, H, T, dims.d_hv, dtype=torch.bfloat16, pin_memory=pin)
    g = Gradients(torch.empty_like(inputs.q, pin_memory=pin), torch.empty_like(inputs.k, pin_memory=pin),
                  torch.empty_like(inputs.v, pin_memory=pin), torch.empty_like(inputs.f_pre, pin_memory=pin),
                  torch.empty_like(inputs.i_pre, pin_memory=pin))
    hin = _ffi.tfla_inputs(inputs.q.data_ptr(), inputs.k.data_ptr(), inputs.v.data_ptr(), inputs.i_pre.data_ptr(),
                           inputs.f_pre.data_ptr())
    gr = _ffi.tfla_grads(g.dq.data_ptr(), g.dk.data_ptr(), g.dv.data_ptr(), g.d_fpre.data_ptr(), g.d_ipre.data_ptr())
    _check(_ffi.lib().tfla_train_step_host(ctypes.byref(dims._c()), int(variant), ctypes.byref(hin), d_h.data_ptr(),
                                           ctypes.byref(gr), h.data_ptr(), _stream()))
    torch.cuda.current_stream().synchronize()
    return h, g


# ---------------------------------------------------------------- split forward entry points
@_on_input_device
def state_recurrence(inputs: SequenceInputs, dims: Dims, variant: Variant, *, all_states: bool = True,
                     keep_saved: bool = True):
    """detail::state_recurrence_head (detail_kernels.hpp:38-44) over every head:
    returns (ChunkStates, saved_states) -- C (fp32, when all_states), n, m and
    the bf16 operand copy C_0..C_{NC-1} (when keep_saved)."""
    dims.validate_chunked()
    inputs.validate(dims)
    if not (all_states or keep_saved):
        raise ParameterError("state_recurrence: request all_states and/or keep_saved")
    dev = inputs.q.device
    B, H, NC = dims.n_batch, dims.n_head, dims.n_chunk()
    f32 = dict(dtype=torch.float32, device=dev)
    C = torch.empty(B, H, NC + 1, dims.d_qk, dims.d_hv, **f32) if all_states else None
    n = torch.empty(B, H, NC + 1, dims.d_qk, **f32)
    m = torch.empty(B, H, NC + 1, **f32)
    saved = (torch.empty(B, H, NC, dims.d_qk, dims.d_hv, dtype=torch.bfloat16, device=dev)
             if keep_saved else None)
    out = _ffi.tfla_fwd_out(None, C.data_ptr() if C is not None else None, n.data_ptr(), m.data_ptr(), None, None,
                            None, None, None, saved.data_ptr() if saved is not None else None)
    ws = _workspace(dims, variant, 0, dev)
    _check(_ffi.lib().tfla_state_recurrence(ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()),
                                            ctypes.byref(out), ws.data_ptr(), ws.numel(), _stream()))
    return ChunkStates(C, n, m), saved


@_on_input_device
def tfla_forward_parallel(inputs: SequenceInputs, dims: Dims, blocks: BlockConfig, variant: Variant,
                          states: ChunkStates, saved_states: Optional[torch.Tensor] = None) -> ChunkwiseForward:
    """detail::tfla_forward_head (tiled.hpp:36-44) over every head: the
    intra-chunk part from materialised states (saved_states, else states.C)."""
    if blocks is None:
        raise ParameterError("tfla_forward_parallel: blocks is required")
    dims.validate_chunked()
    blocks.validate(dims)
    inputs.validate(dims)
    if states is None or (saved_states is None and states.C is None):
        raise ParameterError("tfla_forward_parallel: missing states")
    dev = inputs.q.device
    B, H, T = dims.n_batch, dims.n_head, dims.T
    h = torch.empty(B, H, T, dims.d_hv, dtype=torch.bfloat16, device=dev)
    mc = torch.empty(B, H, T, dtype=torch.float32, device=dev)
    hd = torch.empty(B, H, T, dtype=torch.float32, device=dev)
    ptr = lambda t: t.data_ptr() if t is not None else None
    sin = _ffi.tfla_states_in(ptr(saved_states), ptr(states.C), ptr(states.n), ptr(states.m))
    ws = _workspace(dims, variant, 0, dev)
    _check(_ffi.lib().tfla_forward_parallel(
        ctypes.byref(dims._c()), ctypes.byref(blocks._c()), int(variant), ctypes.byref(inputs._c()),
        ctypes.byref(sin), h.data_ptr(), mc.data_ptr(), hd.data_ptr(), ws.data_ptr(), ws.numel(), _stream()))
    return ChunkwiseForward(h, states, SavedStats(mc, hd), saved_states)


# ---------------------------------------------------------------- split backward entry points
@dataclass
class TfLaDqResult:
    """TfLaDqResult (tiled.hpp:56-59)."""
    dq: torch.Tensor  # bf16 [B,H,T,dqk]
    d_b_cum: torch.Tensor  # fp32 [B,H,T]


@dataclass
class TfLaDkResult:
    """TfLaDkResult (tiled.hpp:64-69)."""
    dk: torch.Tensor  # bf16 [B,H,T,dqk]
    d_a_tail: torch.Tensor  # fp32 [B,H,T]
    d_b_cum: torch.Tensor
    d_i_log: torch.Tensor


@dataclass
class StatePass:
    """backward_state_pass_head outputs (chunkwise.hpp:70-76) for every head."""
    d_c: Optional[torch.Tensor]  # fp32 [B,H,NC+1,dqk,dhv], entry NC is zero
    d_g: torch.Tensor  # fp32 [B,H,NC]


def _split(name: str, inputs, dims, blocks, variant, d_h, states, stats, saved_states, outs):
    if blocks is None:
        raise ParameterError(f"{name}: blocks is required")
    d_h, bin_ = _bwd_in(inputs, dims, d_h, states, stats, blocks, saved_states)
    ws = _workspace(dims, variant, 1, inputs.q.device)
    fn = getattr(_ffi.lib(), name)
    _check(fn(ctypes.byref(dims._c()), ctypes.byref(blocks._c()), int(variant), ctypes.byref(inputs._c()),
              ctypes.byref(bin_), *[o.data_ptr() for o in outs], ws.data_ptr(), ws.numel(), _stream()))


@_on_input_device
def tfla_backward_dq(inputs: SequenceInputs, dims: Dims, blocks: BlockConfig, variant: Variant,
                     d_h: torch.Tensor, states: ChunkStates, stats: SavedStats,
                     saved_states: Optional[torch.Tensor] = None) -> TfLaDqResult:
    """tfla_backward_dq (tiled.hpp:72-74 / tiled.cpp:391-529)."""
    r = TfLaDqResult(torch.empty_like(inputs.q), torch.empty_like(inputs.f_pre))
    _split("tfla_backward_dq", inputs, dims, blocks, variant, d_h, states, stats, saved_states, (r.dq, r.d_b_cum))
    return r


@_on_input_device
def tfla_backward_dk(inputs: SequenceInputs, dims: Dims, blocks: BlockConfig, variant: Variant,
                     d_h: torch.Tensor, states: ChunkStates, stats: SavedStats,
                     saved_states: Optional[torch.Tensor] = None) -> TfLaDkResult:
    """tfla_backward_dk (tiled.hpp:76-79 / tiled.cpp:531-670)."""
    f = inputs.f_pre
    r = TfLaDkResult(torch.empty_like(inputs.k), torch.empty_like(f), torch.empty_like(f), torch.empty_like(f))
    _split("tfla_backward_dk", inputs, dims, blocks, variant, d_h, states, stats, saved_states,
           (r.dk, r.d_a_tail, r.d_b_cum, r.d_i_log))
    return r


@_on_input_device
def tfla_backward_dv(inputs: SequenceInputs, dims: Dims, blocks: BlockConfig, variant: Variant,
                     d_h: torch.Tensor, states: ChunkStates, stats: SavedStats,
                     saved_states: Optional[torch.Tensor] = None) -> torch.Tensor:
    """tfla_backward_dv (tiled.hpp:81-84 / tiled.cpp:672-779)."""
    dv = torch.empty_like(inputs.v)
    _split("tfla_backward_dv", inputs, dims, blocks, variant, d_h, states, stats, saved_states, (dv,))
    return dv


@_on_input_device
def backward_state_pass(inputs: SequenceInputs, dims: Dims, variant: Variant, d_h: torch.Tensor,
                        states: ChunkStates, stats: SavedStats, saved_states: Optional[torch.Tensor] = None,
                        *, with_d_c: bool = True) -> StatePass:
    """detail::backward_state_pass_head (chunkwise.hpp:70-76) over every head."""
    d_h, bin_ = _bwd_in(inputs, dims, d_h, states, stats, None, saved_states)
    dev = inputs.q.device
    B, H, NC = dims.n_batch, dims.n_head, dims.n_chunk()
    d_c = torch.empty(B, H, NC + 1, dims.d_qk, dims.d_hv, dtype=torch.float32, device=dev) if with_d_c else None
    d_g = torch.empty(B, H, NC, dtype=torch.float32, device=dev)
    ws = _workspace(dims, variant, 1, dev)
    _check(_ffi.lib().tfla_backward_state_pass(
        ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()), ctypes.byref(bin_),
        d_c.data_ptr() if d_c is not None else None, d_g.data_ptr(), ws.data_ptr(), ws.numel(), _stream()))
    return StatePass(d_c, d_g)


@_on_input_device
def assemble_gate_grads(inputs: SequenceInputs, dims: Dims, variant: Variant, d_g: torch.Tensor,
                        d_b_total: torch.Tensor, d_a: torch.Tensor, d_i_extra: torch.Tensor):
    """detail::assemble_gate_grads_head (chunkwise.hpp:78-83) over every head;
    returns (d_fpre, d_ipre)."""
    dims.validate_chunked()
    B, H, T, NC = dims.n_batch, dims.n_head, dims.T, dims.n_chunk()
    for name, t, shape in (("d_g", d_g, (B, H, NC)), ("d_b_total", d_b_total, (B, H, T)),
                           ("d_a", d_a, (B, H, T)), ("d_i_extra", d_i_extra, (B, H, T))):
        if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous():
            raise GeometryError(f"assemble_gate_grads: {name} must be contiguous fp32 {shape}")
    dfp = torch.empty_like(inputs.f_pre)
    dip = torch.empty_like(inputs.i_pre)
    _check(_ffi.lib().tfla_assemble_gate_grads(
        ctypes.byref(dims._c()), int(variant), inputs.f_pre.data_ptr(), inputs.i_pre.data_ptr(), d_g.data_ptr(),
        d_b_total.data_ptr(), d_a.data_ptr(), d_i_extra.data_ptr(), dfp.data_ptr(), dip.data_ptr(), _stream()))
    return dfp, dip


# ---------------------------------------------------------------- recurrent (decode) path
@dataclass
class MemoryState:
    """mlstm::MemoryState (core.hpp): C [B,H,dqk,dhv], n [B,H,dqk], m [B,H], fp32 on device."""
    C: torch.Tensor
    n: torch.Tensor
    m: torch.Tensor

    @staticmethod
    def zero(dims: Dims, device="cuda") -> "MemoryState":
        f32 = dict(dtype=torch.float32, device=device)
        B, H = dims.n_batch, dims.n_head
        return MemoryState(torch.zeros(B, H, dims.d_qk, dims.d_hv, **f32), torch.zeros(B, H, dims.d_qk, **f32),
                           torch.zeros(B, H, **f32))

    def clone(self) -> "MemoryState":
        return MemoryState(self.C.clone(), self.n.clone(), self.m.clone())


@dataclass
class RecurrentTrace:
    """mlstm::RecurrentTrace (recurrent.hpp:11-21) without the per-step snapshots."""
    h_tilde: torch.Tensor  # bf16 [B,H,T,dhv]
    C_final: torch.Tensor  # fp32 [B,H,dqk,dhv]
    n_final: torch.Tensor
    m_final: torch.Tensor


@_on_input_device
def recurrent_step(inputs: SequenceInputs, dims: Dims, variant: Variant, state: MemoryState) -> torch.Tensor:
    """Fold step_exp / step_sig (recurrent.cpp:9-63) over dims.T steps, updating
    ``state`` in place (decode). Returns h_tilde bf16 [B,H,T,dhv]."""
    inputs.validate(dims)
    B, H = dims.n_batch, dims.n_head
    for name, t, shape in (("C", state.C, (B, H, dims.d_qk, dims.d_hv)), ("n", state.n, (B, H, dims.d_qk)),
                           ("m", state.m, (B, H))):
        if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous():
            raise GeometryError(f"recurrent_step: state {name} must be contiguous fp32 {shape}")
    h = torch.empty(B, H, dims.T, dims.d_hv, dtype=torch.bfloat16, device=inputs.q.device)
    _check(_ffi.lib().tfla_recurrent_step(
        ctypes.byref(dims._c()), int(variant), ctypes.byref(inputs._c()), state.C.data_ptr(),
        state.n.data_ptr(), state.m.data_ptr(), h.data_ptr(), _stream()))
    return h


@_on_input_device
def run_recurrent(inputs: SequenceInputs, dims: Dims, variant: Variant,
                  initial_state: Optional[MemoryState] = None) -> RecurrentTrace:
    """run_recurrent (recurrent.hpp:42-43; RecurrentOptions::initial_state, :23-27)."""
    st = initial_state.clone() if initial_state is not None else MemoryState.zero(dims, inputs.q.device)
    h = recurrent_step(inputs, dims, Variant(variant), st)
    return RecurrentTrace(h, st.C, st.n, st.m)


@_on_input_device
def output_norm_gate(h_tilde: torch.Tensor, o_pre: torch.Tensor, gamma: torch.Tensor, eps: float = 1e-6,
                     ) -> torch.Tensor:
    """mLSTM cell output (eq. 5): sigmoid(o_pre) * rms_norm(h_tilde; gamma[h], eps),
    rms_norm as transfer.cpp:8-18. h_tilde / o_pre bf16 [B,H,T,dhv], gamma fp32 [H,dhv]."""
    if h_tilde.dim() != 4 or tuple(o_pre.shape) != tuple(h_tilde.shape):
        raise GeometryError("output_norm_gate: h_tilde / o_pre must be [B,H,T,dhv] of the same shape")
    B, H, T, dhv = h_tilde.shape
    if tuple(gamma.shape) != (H, dhv):
        raise GeometryError("output_norm_gate: gamma must be [H, dhv]")
    for name, t, dt in (("h_tilde", h_tilde, torch.bfloat16), ("o_pre", o_pre, torch.bfloat16),
                        ("gamma", gamma, torch.float32)):
        if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise ParameterError(f"{name} must be a contiguous {dt} CUDA tensor")
    h = torch.empty_like(h_tilde)
    dims = Dims(T=T, L=1, d_qk=1, d_hv=dhv, n_head=H, n_batch=B)
    _check(_ffi.lib().tfla_output_norm_gate(ctypes.byref(dims._c()), h_tilde.data_ptr(), o_pre.data_ptr(),
                                            gamma.data_ptr(), float(eps), h.data_ptr(), _stream()))
    return h


@_on_input_device
def apply_gate_softcap(inputs: SequenceInputs, cap: float) -> SequenceInputs:
    """apply_gate_softcap (gates.cpp:61-67): a copy of ``inputs`` with
    i_pre, f_pre <- cap * tanh(x / cap) (softcap, gates.cpp:15-18)."""
    if not cap > 0.0:
        raise ParameterError("softcap: cap must be > 0")
    B, H, T = inputs.i_pre.shape
    io = torch.empty_like(inputs.i_pre)
    fo = torch.empty_like(inputs.f_pre)
    dims = Dims(T=T, L=1, d_qk=1, d_hv=1, n_head=H, n_batch=B)
    _check(_ffi.lib().tfla_apply_gate_softcap(ctypes.byref(dims._c()), inputs.i_pre.data_ptr(),
                                              inputs.f_pre.data_ptr(), float(cap), io.data_ptr(), fo.data_ptr(),
                                              _stream()))
    return SequenceInputs(inputs.q, inputs.k, inputs.v, io, fo)
