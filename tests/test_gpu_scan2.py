"""The TMEM-resident state scan (state_scan2.cu) on both passes: forward (all
C / n states, h) and backward (all gradients, d_g through the assembled
d_fpre) against the f64 oracle, forced on with TFLA_SCAN2=1 (by default it
runs for the forward at L >= 512 only, the measured policy). Tolerances as
everywhere (tests/_util.py)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_H, TOL_STATS, errs, fmt, make_case, np_, to_dev


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape", [(1, 2, 512, 128, 128, 256), (2, 1, 1024, 256, 256, 512), (1, 1, 1024, 512, 128, 512)])
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
def test_scan2_forward_backward_matches_oracle(variant, shape, f_bias, monkeypatch):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    monkeypatch.setenv("TFLA_SCAN2", "1")
    monkeypatch.setenv("TFLA_NO_FUSED_FWD", "1")
    B, H, T, L, dqk, dhv = shape
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=T + L + variant, f_bias=f_bias)
    dh = bf16_round(np.random.default_rng(T + 1).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    f = orc.forward(q, k, v, ip, fp, L, variant)
    g = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    gd = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                            out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    rep = {"h": errs(np_(out.h_tilde), f["h"]), "C": errs(np_(out.states.C), f["C"]),
           "n": errs(np_(out.states.n), f["n"])}
    rep.update({n: errs(np_(getattr(gd, n)), g[n]) for n in ("dq", "dk", "dv", "d_fpre", "d_ipre")})
    print(shape, variant, f_bias, fmt(rep))
    assert rep["h"][0] < TOL_H and rep["C"][0] < TOL_H and rep["n"][0] < TOL_STATS
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rep[n][0] < TOL_GRAD, (n, rep[n])
