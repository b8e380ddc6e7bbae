"""Output epilogue (eq. 5): sigmoid(o) * rms_norm(h_tilde; gamma, eps)
on the B200 kernel vs the f64 oracle restatement (pinned to the reference's
rms_norm, transfer.cpp:8-18, in tests/test_oracle.py). bf16 in / out:
max_rel <= 1e-2."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_H, np_, rel


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(2, 3, 17, 64), (1, 8, 128, 512), (1, 2, 4, 1024)])
@pytest.mark.parametrize("eps", [0.0, 1e-6])
def test_output_norm_gate_matches_oracle(shape, eps):
    import torch

    from paper_2503_14376_b200 import output_norm_gate

    B, H, T, d = shape
    rng = np.random.default_rng(sum(shape))
    x = bf16_round(rng.standard_normal(shape) * 0.3)
    x[0, 0, 0] = 0.0
    o = bf16_round(rng.standard_normal(shape))
    gamma = rng.standard_normal((H, d)).astype(np.float32).astype(np.float64)
    ref = Oracle().output_norm_gate(x, o, gamma, eps)
    bf = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16).contiguous()
    h = output_norm_gate(bf(x), bf(o), torch.from_numpy(gamma).to("cuda", torch.float32).contiguous(), eps)
    torch.cuda.synchronize()
    assert rel(np_(h), ref) < 1e-2
    assert float(h[0, 0, 0].float().abs().max()) == 0.0


@pytest.mark.gpu
def test_gate_softcap_matches_reference_formula():
    """apply_gate_softcap (gates.cpp:61-67) then the forward equals the oracle
    forward on capped pre-activations."""
    import torch

    from paper_2503_14376_b200 import Dims, Variant, apply_gate_softcap, chunkwise_forward
    from tests._util import make_case, to_dev

    B, H, T, L, d = 1, 2, 256, 64, 64
    q, k, v, ip, fp = make_case(B, H, T, d, d, seed=5, gate_scale=8.0)
    cap = 3.0
    capped = apply_gate_softcap(to_dev(q, k, v, ip, fp), cap)
    torch.cuda.synchronize()
    ic, fc = (cap * np.tanh(x / cap) for x in (ip, fp))
    assert np.abs(np_(capped.i_pre) - ic).max() < 1e-6 * cap
    assert np.abs(np_(capped.f_pre) - fc).max() < 1e-6 * cap
    out = chunkwise_forward(capped, Dims(T, L, d, d, H, B), Variant.Exp)
    ref = Oracle().forward(q, k, v, np_(capped.i_pre), np_(capped.f_pre), L, 0)
    assert rel(np_(out.h_tilde), ref["h"]) < TOL_H
    with pytest.raises(Exception):
        apply_gate_softcap(capped, 0.0)


# Gated forward (tfla_chunkwise_forward_gated): forward + output epilogue in
# one call. With TFLA_FUSED_OUT=1 on the fused L = 128 forward the x-tile CTAs
# of a head (a cluster of dhv / 128 CTAs) exchange each row's sum of squares
# over DSMEM; dhv 128 / 256 / 512 give clusters of 1 / 2 / 4, the (8, 8, 1024)
# case runs 256 CTAs = 64 clusters (two waves). Otherwise (default, split
# forward, L != 128) the separate output pass follows the forward.
@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 2, 512, 128, 256, 512), (1, 3, 384, 128, 128, 256),
                                   (2, 1, 256, 128, 128, 128), (8, 8, 1024, 128, 256, 512),
                                   (1, 2, 512, 256, 256, 512)])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("fused_out", [True, False])
def test_forward_gated_matches_separate_pass(shape, variant, fused_out, fwd_path, monkeypatch):
    import torch

    from paper_2503_14376_b200 import (Dims, Variant, chunkwise_forward, chunkwise_forward_gated,
                                       output_norm_gate)
    from tests._util import make_case, to_dev

    B, H, T, L, dqk, dhv = shape
    if fwd_path == "fused" and L != 128:
        pytest.skip("the fused forward is L = 128 only")
    if fused_out:
        monkeypatch.setenv("TFLA_FUSED_OUT", "1")
    else:
        monkeypatch.delenv("TFLA_FUSED_OUT", raising=False)
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=sum(shape) + variant)
    rng = np.random.default_rng(7 + variant)
    o = bf16_round(rng.standard_normal((B, H, T, dhv)))
    gamma = rng.standard_normal((H, dhv)).astype(np.float32)
    inp = to_dev(q, k, v, ip, fp)
    dims = Dims(T, L, dqk, dhv, H, B)
    o_d = torch.from_numpy(o).to("cuda", torch.bfloat16).contiguous()
    g_d = torch.from_numpy(gamma).to("cuda").contiguous()
    eps = 1e-6
    fwd, y = chunkwise_forward_gated(inp, dims, Variant(variant), o_d, g_d, eps)
    plain = chunkwise_forward(inp, dims, Variant(variant))
    y_sep = output_norm_gate(plain.h_tilde, o_d, g_d, eps)
    torch.cuda.synchronize()
    # h_tilde and the saved statistics are exactly the plain forward's
    assert torch.equal(fwd.h_tilde, plain.h_tilde)
    assert torch.equal(fwd.stats.h_denom, plain.stats.h_denom)
    # y: same rms up to fp32 summation order -> at most one bf16 rounding step apart
    d = (y.float() - y_sep.float()).abs()
    assert float(d.max()) <= 2 ** -7 * float(y_sep.float().abs().max())
    assert float((d > 0).float().mean()) < 0.05
    ref = Oracle().output_norm_gate(np_(plain.h_tilde), o, gamma.astype(np.float64), eps)
    assert rel(np_(y), ref) < 1e-2


@pytest.mark.gpu
def test_forward_gated_rejects_bad_arguments():
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward_gated
    from tests._util import make_case, to_dev

    B, H, T, L, d = 1, 2, 256, 128, 128
    inp = to_dev(*make_case(B, H, T, d, d, seed=3))
    dims = Dims(T, L, d, d, H, B)
    o = torch.zeros(B, H, T, d, dtype=torch.bfloat16, device="cuda")
    g = torch.ones(H, d, device="cuda")
    with pytest.raises(Exception):
        chunkwise_forward_gated(inp, dims, Variant.Exp, o, g, -1.0)
    with pytest.raises(Exception):
        chunkwise_forward_gated(inp, dims, Variant.Exp, o, torch.ones(H + 1, d, device="cuda"), 1e-6)
