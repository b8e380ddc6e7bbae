"""CTA-pair (cta_group::2, M = 256) split backward (bwd_pair.cu) for chunks of
L >= 256: dQ / dK / dV and the gate gradients against the f64 oracle, and
against the single-CTA wide kernels on the same inputs. The pair form is
opt-in (TFLA_PAIR_BWD=1; measured no faster, bwd_pair.cu).
Tolerances as everywhere (tests/_util.py)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, errs, fmt, make_case, np_, rel, to_dev

CASES = [
    # B, H, T, L, dqk, dhv
    (1, 2, 512, 256, 256, 256),
    (1, 1, 1024, 512, 256, 512),
    (2, 1, 1024, 256, 256, 512),
    (1, 1, 2048, 1024, 256, 256),
]


def _run(case, variant, f_bias, monkeypatch, pair):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    if pair:
        monkeypatch.setenv("TFLA_PAIR_BWD", "1")
    else:
        monkeypatch.delenv("TFLA_PAIR_BWD", raising=False)
    B, H, T, L, dqk, dhv = case
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=T + L + 3 * variant, f_bias=f_bias)
    dh = bf16_round(np.random.default_rng(T + 5).standard_normal((B, H, T, dhv)))
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    g = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                           out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    return (q, k, v, ip, fp, dh), {n: np_(getattr(g, n)) for n in ("dq", "dk", "dv", "d_fpre", "d_ipre")}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
def test_pair_backward_matches_oracle(case, variant, f_bias, monkeypatch):
    (q, k, v, ip, fp, dh), got = _run(case, variant, f_bias, monkeypatch, pair=True)
    B, H, T, L, dqk, dhv = case
    orc = Oracle()
    f = orc.forward(q, k, v, ip, fp, L, variant)
    ref = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
    rep = {n: errs(got[n], ref[n]) for n in got}
    print(case, variant, f_bias, fmt(rep))
    for n, (e, _, _) in rep.items():
        assert e < TOL_GRAD, (n, e)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_pair_matches_single_cta_kernels(variant, monkeypatch):
    case = (1, 2, 1024, 512, 256, 512)
    _, a = _run(case, variant, 1.0, monkeypatch, pair=True)
    _, b = _run(case, variant, 1.0, monkeypatch, pair=False)
    for n in a:
        assert rel(a[n], b[n]) < 2e-3, n
