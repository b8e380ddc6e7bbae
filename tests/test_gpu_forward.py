"""Forward parity: B200 kernels vs the f64 oracle on identical (bf16 / fp32) inputs.

Tolerance (bf16 tensor-core operands, fp32 accumulation; max_rel = max|x-ref| /
max|ref|, the reference's gradcheck.cpp:7-10 convention; tests/_util.py):
  H, C states, final C      max_rel <= TOL_H (1e-2); per-row <= TOL_ROW on h
  m states / m_combine       exact up to fp32 rounding (abs <= 1e-4 * (1+|ref|))
  h_denom, n states          <= TOL_STATS (1e-2)
max_abs is reported beside max_rel for every tensor.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from tests._util import TOL_H, TOL_ROW, TOL_STATS, errs, fmt, make_case, np_, rel, to_dev

CASES = [
    # B, H, T, L, dqk, dhv
    (1, 2, 256, 64, 64, 64),      # BASELINE config 0 (oracle case)
    (1, 2, 512, 128, 128, 128),
    (2, 1, 512, 256, 128, 256),   # two kv tiles per query tile
    (1, 1, 384, 128, 256, 128),   # d_qk = 256 (two p tiles)
    (1, 1, 192, 64, 64, 128),     # partial last row tile
    (1, 2, 384, 128, 128, 384),   # fused forward, d_qk = 128 (P = 1), three x tiles
    (2, 1, 256, 128, 256, 256),   # fused forward, two x tiles, two heads
]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
def test_forward_matches_oracle(case, variant, f_bias, fwd_path):
    from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward

    B, H, T, L, dqk, dhv = case
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=hash(case) % 1000 + variant, f_bias=f_bias)
    ref = Oracle().forward(q, k, v, ip, fp, L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    out = chunkwise_forward(to_dev(q, k, v, ip, fp), dims, Variant(variant))
    import torch

    torch.cuda.synchronize()
    rep = {
        "h": errs(np_(out.h_tilde), ref["h"]),
        "C": errs(np_(out.states.C), ref["C"]),
        "C_final": errs(np_(out.C_final), ref["C"][:, :, -1]),
        "h_denom": errs(np_(out.stats.h_denom), ref["h_denom"]),
        "n": errs(np_(out.states.n), ref["n"]),
    }
    e = {k_: v[0] for k_, v in rep.items()}
    m_err = np.abs(np_(out.states.m) - ref["m"]) / (1 + np.abs(ref["m"]))
    mc_err = np.abs(np_(out.stats.m_combine) - ref["m_comb"]) / (1 + np.abs(ref["m_comb"]))
    print(case, variant, f_bias, fwd_path, fmt(rep), m_err.max(), mc_err.max())
    assert m_err.max() < 1e-4 and mc_err.max() < 1e-4
    assert e["h"] < TOL_H and e["C"] < TOL_H and e["C_final"] < TOL_H
    assert rep["h"][2] < TOL_ROW
    assert e["h_denom"] < TOL_STATS and e["n"] < TOL_STATS


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_fused_forward_multicast_matches_oracle(variant, monkeypatch):
    """Opt-in cluster variant of K12 (TFLA_FWD_MULTICAST=1): the 4 x-tile CTAs of
    a head share the Q/K stages by TMA multicast; same results as the oracle."""
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward

    monkeypatch.setenv("TFLA_FORCE_FUSED_FWD", "1")
    monkeypatch.setenv("TFLA_FWD_MULTICAST", "1")
    B, H, T, L, dqk, dhv = 1, 2, 512, 128, 256, 512
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=61 + variant)
    ref = Oracle().forward(q, k, v, ip, fp, L, variant)
    out = chunkwise_forward(to_dev(q, k, v, ip, fp), Dims(T, L, dqk, dhv, H, B), Variant(variant))
    torch.cuda.synchronize()
    assert rel(np_(out.h_tilde), ref["h"]) < TOL_H
    assert rel(np_(out.states.C), ref["C"]) < TOL_H
