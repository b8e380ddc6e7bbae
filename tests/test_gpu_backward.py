"""Backward parity: B200 kernels vs the f64 oracle (chunkwise_backward semantics:
normaliser and max states detached, chunkwise.cpp:396-566).

Tolerance (bf16 tensor-core operands incl. bf16 dH and bf16 saved states, fp32
accumulation; max_rel = max|x-ref| / max|ref|, gradcheck.cpp:7-10):
  dq, dk, dv, d_fpre, d_ipre max_rel <= TOL_GRAD (1.5e-2, tests/_util.py);
  per-row (dq, dk, dv rows) <= TOL_ROW; max_abs reported beside max_rel
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_ROW, errs, fmt, make_case, np_, rel, to_dev

CASES = [
    # B, H, T, L, dqk, dhv
    (1, 2, 256, 64, 64, 64),
    (1, 2, 512, 128, 128, 128),
    (2, 1, 512, 256, 128, 256),
    (1, 1, 384, 128, 256, 128),
    (1, 1, 192, 64, 64, 128),
    (1, 2, 384, 128, 256, 256),   # fused backward with two dV tiles, two p tiles
    (1, 1, 256, 128, 128, 384),   # fused backward, d_qk = 128, three dV tiles
]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
@pytest.mark.parametrize("from_fp32_states", [False, True])
def test_backward_matches_oracle(case, variant, f_bias, from_fp32_states, fwd_path):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    B, H, T, L, dqk, dhv = case
    seed = hash(case) % 1000 + 17 * variant
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=seed, f_bias=f_bias)
    dh = bf16_round(np.random.default_rng(seed + 1).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    fwd = orc.forward(q, k, v, ip, fp, L, variant)
    ref = orc.backward(q, k, v, ip, fp, dh, fwd["C"], fwd["m"], fwd["m_comb"], fwd["h_denom"], L, variant)

    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    dh_t = torch.from_numpy(dh).to("cuda", torch.bfloat16)
    g = chunkwise_backward(inp, dims, Variant(variant), dh_t, out.states, out.stats,
                           saved_states=None if from_fp32_states else out.saved_states)
    torch.cuda.synchronize()
    rep = {n: errs(np_(getattr(g, n)), ref[n]) for n in ("dq", "dk", "dv", "d_fpre", "d_ipre")}
    print(case, variant, f_bias, from_fp32_states, fmt(rep))
    for n, (e, _, row) in rep.items():
        assert e < TOL_GRAD, (n, e)
        if n in ("dq", "dk", "dv"):
            assert row < TOL_ROW, (n, row)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_dg_identity_mode_within_tolerance(variant, monkeypatch):
    """TFLA_DG_IDENTITY=1 (d_g from per-token partials, no state reads in the
    scan) stays within the backward tolerance; dq/dk/dv are unchanged."""
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    B, H, T, L, dqk, dhv = 1, 2, 512, 128, 256, 256
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=71 + variant, f_bias=3.0)
    dh = bf16_round(np.random.default_rng(72).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    fwd = orc.forward(q, k, v, ip, fp, L, variant)
    ref = orc.backward(q, k, v, ip, fp, dh, fwd["C"], fwd["m"], fwd["m_comb"], fwd["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    dh_t = torch.from_numpy(dh).to("cuda", torch.bfloat16)
    direct = chunkwise_backward(inp, dims, Variant(variant), dh_t, out.states, out.stats, out.saved_states)
    monkeypatch.setenv("TFLA_DG_IDENTITY", "1")
    ident = chunkwise_backward(inp, dims, Variant(variant), dh_t, out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    for n in ("dq", "dk", "dv", "d_ipre"):
        assert torch.equal(getattr(direct, n), getattr(ident, n)), n
    assert rel(np_(ident.d_fpre), ref["d_fpre"]) < 3e-2


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
def test_wide_fused_backward_matches_oracle(variant, f_bias, monkeypatch):
    """The opt-in 256-column-group fused backward (bwd_fused_wide.cu,
    TFLA_WIDE_FUSED_BWD=1) against the oracle at the 7B head geometry."""
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    monkeypatch.setenv("TFLA_WIDE_FUSED_BWD", "1")
    B, H, T, L, dqk, dhv = 1, 2, 512, 128, 256, 512
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=91 + variant, f_bias=f_bias)
    dh = bf16_round(np.random.default_rng(92).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    fwd = orc.forward(q, k, v, ip, fp, L, variant)
    ref = orc.backward(q, k, v, ip, fp, dh, fwd["C"], fwd["m"], fwd["m_comb"], fwd["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    g = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                           out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rel(np_(getattr(g, n)), ref[n]) < TOL_GRAD, n
