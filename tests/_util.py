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
