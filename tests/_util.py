"""Shared helpers for the parity tests (test infrastructure)."""
import numpy as np

from oracle.oracle import bf16_round


def make_case(B, H, T, dqk, dhv, seed, f_bias=0.0, gate_scale=1.0):
    """Seeded inputs: q,k,v ~ N(0,1) rounded to bf16; i,f ~ gate_scale*N(0,1)
    (+ f_bias) rounded to fp32 -- the values both sides see exactly."""
    rng = np.random.default_rng(seed)
    q = bf16_round(rng.standard_normal((B, H, T, dqk)))
    k = bf16_round(rng.standard_normal((B, H, T, dqk)))
    v = bf16_round(rng.standard_normal((B, H, T, dhv)))
    ip = (gate_scale * rng.standard_normal((B, H, T))).astype(np.float32).astype(np.float64)
    fp = (gate_scale * rng.standard_normal((B, H, T)) + f_bias).astype(np.float32).astype(np.float64)
    return q, k, v, ip, fp


def to_dev(q, k, v, ip, fp):
    import torch

    from paper_2503_14376_b200 import SequenceInputs

    bf = lambda a: torch.from_numpy(a).to(device="cuda", dtype=torch.bfloat16).contiguous()
    f32 = lambda a: torch.from_numpy(a).to(device="cuda", dtype=torch.float32).contiguous()
    return SequenceInputs(bf(q), bf(k), bf(v), f32(ip), f32(fp))


def rel(a, ref):
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(float(np.abs(ref).max()), 1e-12)
    return float(np.abs(a - ref).max()) / scale


def np_(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


# Parity tolerances (bf16 tensor-core operands, fp32 accumulation), stated once
# for every GPU-vs-oracle test; max_rel = max|x - ref| / max|ref| (the
# reference's gradcheck.cpp:7-10 convention). Observed on B200: h 2-5e-3,
# C 1-3e-3, gradients 2-7e-3.
TOL_H = 1e-2       # h, C states, C_final
TOL_STATS = 1e-2   # h_denom, n states
TOL_GRAD = 1.5e-2  # dq, dk, dv, d_fpre, d_ipre
# Per-row check (rows = last axis): on rows whose reference max is at least
# ROW_FLOOR of the tensor max, max|dx| / max|ref row| <= TOL_ROW -- a
# global-max normaliser alone would hide errors on low-magnitude rows.
ROW_FLOOR = 1e-2
TOL_ROW = 6e-2


def errs(a, ref):
    """(max_rel, max_abs, worst per-row relative error) of a vs ref."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.abs(a - ref)
    gmax = max(float(np.abs(ref).max()), 1e-30)
    row_ref = np.abs(ref).max(axis=-1)
    row_err = d.max(axis=-1)
    keep = row_ref >= ROW_FLOOR * gmax
    row_rel = float((row_err[keep] / row_ref[keep]).max()) if keep.any() else 0.0
    return float(d.max()) / gmax, float(d.max()), row_rel


def fmt(report):
    return {k: f"rel {v[0]:.2e} abs {v[1]:.2e} row {v[2]:.2e}" for k, v in report.items()}
