"""Closed-form cost model of the chunkwise formulation (the reference's
perfmodel, perfmodel.hpp / perfmodel.cpp), used as the roofline reporter of
bench.py with the MEASURED B200 peaks (MEASURED_PEAKS.json) in place of the
reference's nominal "B200 HGX" preset (perfmodel.cpp:277-285).

Host-side arithmetic only (no device work). Every function restates the
reference formula it cites; tests/test_perfmodel.py pins them against the
reference library built from its own sources.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import Callable, Dict, List, Optional, Sequence

from .mlstm import Dims, GeometryError, ParameterError, Variant

EXP, SIG = Variant.Exp, Variant.Sig


@dataclass(frozen=True)
class PerfParams:
    """PerfParams (perfmodel.hpp:16-24): causal fraction, per-op weights and
    storage widths (bf16 activations, fp32 states by default)."""
    f_causal: float = 0.5
    f_exp: float = 1.0
    f_log: float = 1.0
    f_sig: float = 1.0
    f_max: float = 1.0
    f_abs: float = 1.0
    f_mask: float = 1.0
    bytes_qkv: float = 2.0
    bytes_if: float = 2.0
    bytes_cmn: float = 4.0

    def validate(self) -> None:  # perfmodel.cpp:11-17
        if not 0.5 <= self.f_causal <= 1.0:
            raise ParameterError("f_causal must lie in [0.5, 1]")
        if any(b not in (2.0, 4.0) for b in (self.bytes_qkv, self.bytes_if, self.bytes_cmn)):
            raise ParameterError("byte widths must be 2 or 4")

    def simplified(self) -> "PerfParams":  # perfmodel.cpp:19-23
        return replace(self, f_exp=1.0, f_log=1.0, f_sig=1.0, f_max=1.0, f_abs=1.0, f_mask=1.0)


@dataclass(frozen=True)
class AcceleratorSpec:
    """AcceleratorSpec (perfmodel.hpp:26-30)."""
    name: str
    flops_per_s: float
    bytes_per_s: float


@dataclass
class CostBreakdown:
    """CostBreakdown (perfmodel.hpp:38-44): named FLOP line items."""
    items: List[tuple] = field(default_factory=list)

    def total(self) -> float:
        return sum(v for _, v in self.items)

    def item(self, name: str) -> float:
        for n, v in self.items:
            if n == name:
                return v
        raise ParameterError(f"unknown cost item: {name}")


@dataclass
class MemopCounts:
    loaded: float = 0.0
    stored: float = 0.0

    def total(self) -> float:
        return self.loaded + self.stored


def _validate_chunked(dims: Dims) -> None:
    """Dims::validate_chunked (core.cpp:9-21) -- the model's own rule, not the
    kernels' tile constraints (the model is evaluated at any geometry)."""
    if min(dims.n_batch, dims.n_head, dims.T, dims.L, dims.d_qk, dims.d_hv) < 1:
        raise GeometryError("dims must be positive")
    if dims.T % dims.L:
        raise GeometryError("T must be a multiple of the chunk size L")


def _prep(params: PerfParams, simplified: bool) -> PerfParams:
    params.validate()
    return params.simplified() if simplified else params


def flops_chunkwise(dims: Dims, params: PerfParams, variant: Variant, simplified: bool = False) -> CostBreakdown:
    """flops_chunkwise (perfmodel.cpp:52-98): per-chunk items x B*H*NC."""
    _validate_chunked(dims)
    p = _prep(params, simplified)
    L, dqk, dhv, fc = float(dims.L), float(dims.d_qk), float(dims.d_hv), p.f_causal
    scale = float(dims.n_batch * dims.n_head * dims.n_chunk())
    tri = 0.5 * L * (L + 1.0)
    if Variant(variant) == EXP:
        gates = 2 * L + tri + L * (1 + p.f_exp + p.f_log + p.f_sig) + 3 + p.f_max + p.f_exp
        denominator = 2 * dqk + 2 * L * dqk
        cum_forget = tri + L * (p.f_log + p.f_sig)
        gate_matrix = fc * (L * L * (3 + p.f_exp + p.f_max) + L * (1 + p.f_max))
        inter = 2 * L * dqk * dhv + 3 * L * dqk
        combination = 2 * L * dhv + L * (1 + p.f_max + p.f_abs + p.f_exp)
    else:
        gates = 2 * L + tri + L * p.f_exp + p.f_exp + 2 * L * (p.f_log + p.f_sig)
        denominator = 0.0
        cum_forget = tri + 2 * L * (p.f_log + p.f_sig)
        gate_matrix = fc * (L * L * (2 + p.f_exp))
        inter = 2 * L * dqk * dhv + L * dqk
        combination = L * dhv
    numerator = 2 * dqk * dhv + 2 * L * dqk * dhv + L * dqk
    intra = fc * (2 * L * L * (dqk + dhv) + 3 * L * L)
    names = ("gates", "numerator", "denominator", "cum_forget", "gate_matrix", "intra_outputs",
             "inter_outputs", "combination")
    vals = (gates, numerator, denominator, cum_forget, gate_matrix, intra, inter, combination)
    return CostBreakdown([(n, scale * v) for n, v in zip(names, vals)])


def flops_parallel(dims: Dims, params: PerfParams, variant: Variant, simplified: bool = False) -> CostBreakdown:
    """flops_parallel (perfmodel.cpp:100-126)."""
    p = _prep(params, simplified)
    T, dqk, dhv, fc = float(dims.T), float(dims.d_qk), float(dims.d_hv), p.f_causal
    scale = float(dims.n_batch * dims.n_head)
    is_exp = Variant(variant) == EXP
    cum_forget = 0.5 * T * (T + 1) + (T * (p.f_log + p.f_sig) if is_exp else 2 * T * (p.f_log + p.f_sig))
    gate_matrix = T * T * (3 + p.f_exp + p.f_max + p.f_mask)
    logits = fc * (2 * T * T * dqk + 2 * T * T)
    norm = fc * (T * T * (3 + p.f_abs) + T * (p.f_exp + p.f_max)) if is_exp else 0.0
    outputs = fc * 2 * T * T * dhv
    return CostBreakdown([("cum_forget", scale * cum_forget), ("gate_matrix", scale * gate_matrix),
                          ("attention_logits", scale * logits), ("normalization", scale * norm),
                          ("outputs", scale * outputs)])


def flops_recurrent(dims: Dims, params: PerfParams, variant: Variant, simplified: bool = False) -> CostBreakdown:
    """flops_recurrent (perfmodel.cpp:128-154)."""
    p = _prep(params, simplified)
    dqk, dhv = float(dims.d_qk), float(dims.d_hv)
    scale = float(dims.n_batch * dims.n_head) * float(dims.T)
    if Variant(variant) == EXP:
        gates = 4 + 2 * p.f_exp + p.f_log + p.f_sig + p.f_max
        den = 6 * dqk + dhv + 1 + p.f_abs + p.f_max
    else:
        gates, den = 2 * p.f_sig, 0.0
    return CostBreakdown([("gates", scale * gates), ("memory_cell_update", scale * 4 * dqk * dhv),
                          ("denominator_scale", scale * den), ("output", scale * (2 * dqk * dhv + dqk))])


def memops(dims: Dims, params: PerfParams, variant: Variant, formulation: str) -> MemopCounts:
    """memops (perfmodel.cpp:156-195): bytes loaded / stored per formulation."""
    params.validate()
    dqk, dhv = float(dims.d_qk), float(dims.d_hv)
    bq, bi, bc = params.bytes_qkv, params.bytes_if, params.bytes_cmn
    is_exp = Variant(variant) == EXP
    state = dqk * dhv + dqk + 1 if is_exp else dqk * dhv
    if formulation == "chunkwise":
        _validate_chunked(dims)
        L = float(dims.L)
        scale = float(dims.n_batch * dims.n_head * dims.n_chunk())
        load = L * (dqk + dhv) * bq + 2 * L * bi + L * (2 * dqk + dhv) * bq + 2 * L * bi + state * bc
        store = state * bc + L * dhv * bq + (2 * L * bc if is_exp else 0.0)
        return MemopCounts(scale * load, scale * store)
    if formulation == "parallel":
        T = float(dims.T)
        scale = float(dims.n_batch * dims.n_head)
        return MemopCounts(scale * (T * (2 * dqk + dhv) * bq + 2 * T * bi),
                           scale * (T * dhv * bq + (2 * T * bc if is_exp else 0.0)))
    if formulation == "recurrent":
        scale = float(dims.n_batch * dims.n_head) * float(dims.T)
        return MemopCounts(scale * ((2 * dqk + dhv) * bq + 2 * bi + state * bc), scale * (dhv * bq + state * bc))
    raise ParameterError(f"unknown formulation: {formulation}")


def chunkwise_flops_model(variant: Variant, T: float, L: float, d_qk: float, d_hv: float, f_causal: float) -> float:
    """Closed-form FLOPs per head (perfmodel.cpp:199-209)."""
    dd = d_qk * d_hv
    if Variant(variant) == SIG:
        return (T * L * f_causal * (2 * (d_qk + d_hv) + 6) + T * L + T * (4 * dd + 2 * d_qk + d_hv + 11)
                + (T / L) * (2 * dd + 5))
    return (T * L * f_causal * (2 * (d_qk + d_hv) + 8) + T * L + 2 * T * f_causal
            + T * (4 * dd + 6 * d_qk + 4 * d_hv + 13) + (T / L) * (2 * dd + 2 * d_qk + 5))


def chunkwise_bytes_model(variant: Variant, T: float, L: float, d_qk: float, d_hv: float, params: PerfParams) -> float:
    """Closed-form bytes per head (perfmodel.cpp:211-219)."""
    state = L + d_hv * d_qk + d_qk + 1 if Variant(variant) == EXP else d_hv * d_qk
    per_chunk = 4 * L * params.bytes_if + 3 * L * (d_hv + d_qk) * params.bytes_qkv + 2 * state * params.bytes_cmn
    return (T / L) * per_chunk


def flop_optimal_chunk_size(d_hv: float, p_qk: float, f_causal: float) -> float:
    """perfmodel.cpp:221-227."""
    if d_hv <= 0 or p_qk <= 0 or f_causal <= 0:
        raise ParameterError("flop_optimal_chunk_size: arguments must be positive")
    return math.sqrt((2 * d_hv * d_hv * p_qk + 5) / (2 * f_causal * (d_hv * (1 + p_qk) + 3) + 1))


def runtime_optimal_chunk_size(d_hv: float, p_qk: float, f_causal: float, bytes_cmn: float, i_acc: float) -> float:
    """perfmodel.cpp:229-237."""
    if d_hv <= 0 or p_qk <= 0 or f_causal <= 0 or bytes_cmn <= 0 or i_acc < 0:
        raise ParameterError("runtime_optimal_chunk_size: arguments must be positive")
    num = 2 * d_hv * d_hv * p_qk + 5 + 2 * i_acc * d_hv * d_hv * p_qk * bytes_cmn
    return math.sqrt(num / (2 * f_causal * (d_hv * (1 + p_qk) + 3) + 1))


def theoretical_runtime(dims: Dims, params: PerfParams, variant: Variant, accel: AcceleratorSpec, L: float,
                        bound: str = "max") -> float:
    """Modelled forward seconds, FLOP time + / max memory time (perfmodel.cpp:239-256)."""
    if L < 1:
        raise ParameterError("theoretical_runtime: L must be >= 1")
    if accel.flops_per_s <= 0 or accel.bytes_per_s <= 0:
        raise ParameterError("theoretical_runtime: accelerator rates must be positive")
    scale = float(dims.n_batch * dims.n_head)
    args = (variant, float(dims.T), float(L), float(dims.d_qk), float(dims.d_hv))
    t_f = scale * chunkwise_flops_model(*args, params.f_causal) / accel.flops_per_s
    t_b = scale * chunkwise_bytes_model(*args, params) / accel.bytes_per_s
    return t_f + t_b if bound == "sum" else max(t_f, t_b)


def arithmetic_intensity(dims: Dims, params: PerfParams, L: float) -> float:
    """FLOP/byte of the sigmoid forward (perfmodel.cpp:258-266)."""
    if L < 1:
        raise ParameterError("arithmetic_intensity: L must be >= 1")
    a = (SIG, float(dims.T), float(L), float(dims.d_qk), float(dims.d_hv))
    return chunkwise_flops_model(*a, params.f_causal) / chunkwise_bytes_model(*a, params)


def accelerator_intensity(accel: AcceleratorSpec) -> float:
    if accel.bytes_per_s <= 0:
        raise ParameterError("accelerator bandwidth must be positive")
    return accel.flops_per_s / accel.bytes_per_s


def roofline(accel: AcceleratorSpec, intensity: float) -> float:
    """min(bandwidth x intensity, peak) (perfmodel.cpp:273-276)."""
    if intensity < 0:
        raise ParameterError("roofline: intensity must be >= 0")
    return min(accel.bytes_per_s * intensity, accel.flops_per_s)


# perfmodel.cpp:277-285 (nominal datasheet presets)
PRESETS = (AcceleratorSpec("V100 SXM2", 120e12, 0.9e12), AcceleratorSpec("A100 SXM", 312e12, 1.935e12),
           AcceleratorSpec("H100 SXM", 989e12, 3.35e12), AcceleratorSpec("B200 HGX", 2250e12, 7.7e12))


def measured_b200(path: Optional[Path] = None, sustained: bool = False) -> AcceleratorSpec:
    """The B200 of this pool as measured by the driver (MEASURED_PEAKS.json):
    copy bandwidth and cuBLAS bf16 throughput (burst, or sustained)."""
    path = Path(path or Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json")
    if not path.exists():  # the profiling recipe's stated fallback (bench.py peaks())
        tf = 1400.0 if sustained else 1590.0
        return AcceleratorSpec("B200 fallback" + (" sustained" if sustained else ""), tf * 1e12, 6650.0e9)
    pk = json.loads(path.read_text())
    tf = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) if sustained else pk["bf16_tflops"]
    return AcceleratorSpec("B200 measured" + (" sustained" if sustained else ""), tf * 1e12, pk["hbm_gbs"] * 1e9)


def load_accelerator_file(path) -> List[AcceleratorSpec]:
    """JSON array of {name, flops_per_s, bytes_per_s} (perfmodel.cpp:287-304)."""
    j = json.loads(Path(path).read_text())
    if not isinstance(j, list):
        raise ParameterError("accelerator file must hold a JSON array")
    out = []
    for e in j:
        a = AcceleratorSpec(str(e["name"]), float(e["flops_per_s"]), float(e["bytes_per_s"]))
        if a.flops_per_s <= 0 or a.bytes_per_s <= 0:
            raise ParameterError(f"accelerator rates must be positive: {a.name}")
        out.append(a)
    return out


def find_accelerator(name: str, extra: Sequence[AcceleratorSpec] = ()) -> AcceleratorSpec:
    for a in list(extra) + list(PRESETS):
        if a.name == name:
            return a
    raise ParameterError(f"unknown accelerator: {name}")


def chunk_size_candidates(lo: int, hi: int, T: int) -> List[int]:
    """Divisors of T in [lo, hi] (T > 0), else every integer (perfmodel.cpp:315-330)."""
    if lo < 1 or hi < lo:
        raise ParameterError("invalid chunk-size range")
    out = [l for l in range(lo, min(hi, T) + 1) if T % l == 0] if T > 0 else list(range(lo, hi + 1))
    if not out:
        raise ParameterError("no chunk-size candidates in range")
    return out


def _argmin(cands: Sequence[int], fn: Callable[[int], float]) -> int:
    best, best_v = cands[0], math.inf
    for l in cands:
        v = fn(l)
        if v < best_v:
            best, best_v = l, v
    return best


def flop_argmin_chunk_size(d_hv: float, p_qk: float, f_causal: float, candidates: Sequence[int]) -> int:
    """perfmodel.cpp:345-353 (T = 8192 scaling constant)."""
    d_qk = p_qk * d_hv
    return _argmin(candidates, lambda l: chunkwise_flops_model(SIG, 8192.0, float(l), d_qk, d_hv, f_causal))


def runtime_argmin_chunk_size(d_hv: float, p_qk: float, f_causal: float, bytes_cmn: float, accel: AcceleratorSpec,
                              candidates: Sequence[int]) -> int:
    """perfmodel.cpp:355-367: argmin of the sum-bound sigmoid runtime (T = 8192 constant)."""
    params = PerfParams(f_causal=f_causal, bytes_cmn=bytes_cmn)
    d_qk = p_qk * d_hv

    def rt(l):
        a = (SIG, 8192.0, float(l), d_qk, d_hv)
        return (chunkwise_flops_model(*a, f_causal) / accel.flops_per_s
                + chunkwise_bytes_model(*a, params) / accel.bytes_per_s)

    return _argmin(candidates, rt)


def report(dims: Dims, variant: Variant, accel: AcceleratorSpec, params: PerfParams = PerfParams()) -> Dict:
    """The reference's modelled forward at dims.L on `accel` plus the chunk
    sizes its closed forms call optimal: the roofline line bench.py prints."""
    i_acc = accelerator_intensity(accel)
    p_qk = dims.d_qk / dims.d_hv
    return {
        "accelerator": accel.name,
        "flops_per_s": accel.flops_per_s,
        "bytes_per_s": accel.bytes_per_s,
        "fwd_model_ms_max": 1e3 * theoretical_runtime(dims, params, variant, accel, dims.L, "max"),
        "fwd_model_ms_sum": 1e3 * theoretical_runtime(dims, params, variant, accel, dims.L, "sum"),
        "intensity_flop_per_byte": arithmetic_intensity(dims, params, dims.L),
        "accelerator_intensity": i_acc,
        "flop_optimal_L": flop_optimal_chunk_size(dims.d_hv, p_qk, params.f_causal),
        "runtime_optimal_L": runtime_optimal_chunk_size(dims.d_hv, p_qk, params.f_causal, params.bytes_cmn, i_acc),
    }
