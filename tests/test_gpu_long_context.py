"""Long context (BASELINE configs[3]: B=1, NH=8, S=65536, dqk=256, dhv=512):
forward and backward parity on the full chain length.

At L=128 a head walks 512 chunks (L=512: 128), with the bf16 operand copy of
every state feeding the backward; error accumulation along chains 8x longer
than the 7B shape's is what this checks. Two heads (the f64 oracle runs one
host thread per head) at the exact BASELINE head geometry and length; every
output -- h, the final C / n / m, m_comb, h_denom and all five gradients --
against the oracle, on the default (split) forward and the forced fused one.
Tolerances as everywhere (tests/_util.py): h, C <= TOL_H, gradients <= TOL_GRAD.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_H, TOL_STATS, errs, fmt, make_case, np_, to_dev

B, H, T, DQK, DHV = 1, 2, 65536, 256, 512
_CACHE = {}


def _oracle(variant, L, f_bias):
    key = (variant, L, f_bias)
    if key not in _CACHE:
        q, k, v, ip, fp = make_case(B, H, T, DQK, DHV, seed=650 + 7 * variant + L, f_bias=f_bias)
        dh = bf16_round(np.random.default_rng(651 + L).standard_normal((B, H, T, DHV)))
        orc = Oracle()
        orc.threads = H
        f = orc.forward(q, k, v, ip, fp, L, variant)
        g = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
        ref = {"h": f["h"], "C_final": f["C"][:, :, -1].copy(), "n_final": f["n"][:, :, -1].copy(),
               "m": f["m"], "m_comb": f["m_comb"], "h_denom": f["h_denom"], **g}
        del f
        _CACHE.clear()  # one reference set alive at a time (the f64 states are ~1 GB)
        _CACHE[key] = ((q, k, v, ip, fp, dh), ref)
    return _CACHE[key]


@pytest.mark.gpu
@pytest.mark.parametrize("variant,L,f_bias", [(0, 128, 0.0), (1, 512, 3.0), (0, 512, 3.0)])
def test_long_context_matches_oracle(variant, L, f_bias, fwd_path):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    if fwd_path == "fused" and L != 128:
        pytest.skip("the fused forward is the L=128 kernel")
    (q, k, v, ip, fp, dh), ref = _oracle(variant, L, f_bias)
    dims = Dims(T=T, L=L, d_qk=DQK, d_hv=DHV, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant), all_states=False)
    g = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                           out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    rep = {"h": errs(np_(out.h_tilde), ref["h"]), "C_final": errs(np_(out.C_final), ref["C_final"]),
           "h_denom": errs(np_(out.stats.h_denom), ref["h_denom"])}
    if variant == 0:
        rep["n_final"] = errs(np_(out.n_final), ref["n_final"])
    rep.update({n: errs(np_(getattr(g, n)), ref[n]) for n in ("dq", "dk", "dv", "d_fpre", "d_ipre")})
    m_err = np.abs(np_(out.states.m) - ref["m"]) / (1 + np.abs(ref["m"]))
    mc_err = np.abs(np_(out.stats.m_combine) - ref["m_comb"]) / (1 + np.abs(ref["m_comb"]))
    print(f"S={T} L={L} variant={variant} f_bias={f_bias} {fwd_path}:", fmt(rep), m_err.max(), mc_err.max())
    assert m_err.max() < 1e-4 and mc_err.max() < 1e-4
    assert rep["h"][0] < TOL_H and rep["C_final"][0] < TOL_H
    assert rep["h_denom"][0] < TOL_STATS and rep.get("n_final", (0,))[0] < TOL_STATS
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rep[n][0] < TOL_GRAD, (n, rep[n])
