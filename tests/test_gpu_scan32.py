"""32-column state-scan tiles (K1 / K3, opt-in TFLA_SCAN32=1: 64-byte swizzled
B / state / C_k tiles, N = 32 MMAs, two CTAs per SM) vs the f64 oracle on the
split forward (C, n states, h) and the backward (all five gradients, whose d_g
partials come from K3's C_k . dC_{k+1} dots). Tolerances as
tests/test_gpu_forward.py / tests/test_gpu_backward.py."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_H, make_case, np_, rel, to_dev

CASES = [
    # B, H, T, L, dqk, dhv
    (1, 2, 512, 128, 256, 512),
    (1, 1, 384, 128, 128, 64),
    (2, 1, 512, 256, 64, 128),
]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
def test_scan32_forward_backward_match_oracle(case, variant, f_bias, monkeypatch):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    monkeypatch.setenv("TFLA_SCAN32", "1")
    monkeypatch.setenv("TFLA_NO_FUSED_FWD", "1")
    monkeypatch.delenv("TFLA_FORCE_FUSED_FWD", raising=False)
    B, H, T, L, dqk, dhv = case
    seed = hash(case) % 1000 + 31 * variant
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=seed, f_bias=f_bias)
    dh = bf16_round(np.random.default_rng(seed + 1).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    ref = orc.forward(q, k, v, ip, fp, L, variant)
    rg = orc.backward(q, k, v, ip, fp, dh, ref["C"], ref["m"], ref["m_comb"], ref["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    g = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                           out.states, out.stats, saved_states=out.saved_states)
    torch.cuda.synchronize()
    assert rel(np_(out.states.C), ref["C"]) < TOL_H
    assert rel(np_(out.states.n), ref["n"]) < 1e-2
    assert rel(np_(out.h_tilde), ref["h"]) < TOL_H
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rel(np_(getattr(g, n)), rg[n]) < TOL_GRAD, n
