"""chunkwise_forward_frozen on the B200 kernels (chunkwise.cpp:304-394) and a
finite-difference check of the GPU backward against it.

The reference's backward is the exact gradient of the frozen forward (max
states, m_comb and h_denom pinned, chunkwise.hpp:42-54); its FD oracle
differentiates that function (gradcheck.cpp:31-64, acceptance criterion 2,
acceptance.cpp:84). Here both sides are the GPU library:
  * frozen(live stats) == live forward (test_chunkwise.cpp:177-186), within
    the bf16-operand tolerance (the two run different kernel paths);
  * directional derivatives: for L(x) = sum(w * h_frozen(x)) and the GPU
    gradient g = chunkwise_backward(dH = w), central differences
    (L(x + d+) - L(x + d-)) match <g, d+ - d-> for q, k, v, i_pre, f_pre.
    h_frozen is linear in each of q, k, v (the pinned stats remove every
    nonlinearity), so those differences are exact at any step; d+/- are the
    actually representable bf16 perturbations. The gates enter through exp:
    fp32 perturbations of 2e-2 along sign(g) * U(0.5, 1.5) keep the O(eps^2)
    and the bf16 h-rounding noise below 1%. Tolerance 3% relative.
"""
import numpy as np
import pytest

from tests._util import make_case, np_, rel, to_dev


def _setup(variant, L, seed=5, B=1, H=2, T=256, dqk=64, dhv=64, f_bias=0.0):
    import torch

    from paper_2503_14376_b200 import Dims, SequenceInputs, Variant, chunkwise_backward, chunkwise_forward

    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed, f_bias=f_bias)
    inp = to_dev(q, k, v, ip, fp)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    out = chunkwise_forward(inp, dims, Variant(variant))
    w = torch.randn(B, H, T, dhv, device="cuda", generator=torch.Generator("cuda").manual_seed(seed)).to(torch.bfloat16)
    g = chunkwise_backward(inp, dims, Variant(variant), w, out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    return inp, dims, out, w, g


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("L", [64, 128, 256])
def test_frozen_equals_live_forward(variant, L, fwd_path):
    from paper_2503_14376_b200 import Variant, chunkwise_forward_frozen

    inp, dims, out, _, _ = _setup(variant, L, T=512, dqk=128, dhv=128, f_bias=1.0)
    hf = chunkwise_forward_frozen(inp, dims, Variant(variant), out.states, out.stats)
    e = rel(np_(hf), np_(out.h_tilde))
    print(f"variant={variant} L={L} frozen vs live max_rel={e:.2e}")
    assert e < 1e-2


@pytest.mark.gpu
def test_frozen_requires_saved_stats():
    from paper_2503_14376_b200 import ChunkStates, ParameterError, Variant, chunkwise_forward_frozen

    inp, dims, out, _, _ = _setup(0, 64)
    with pytest.raises(ParameterError):
        chunkwise_forward_frozen(inp, dims, Variant.Exp, ChunkStates(None, None, None), out.stats)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("L", [64, 128])
def test_backward_matches_directional_derivatives(variant, L):
    import torch

    from paper_2503_14376_b200 import SequenceInputs, Variant, chunkwise_forward_frozen

    inp, dims, out, w, g = _setup(variant, L)
    wd = w.double()
    gen = torch.Generator("cuda").manual_seed(99 + variant)

    def loss(x: SequenceInputs) -> float:
        h = chunkwise_forward_frozen(x, dims, Variant(variant), out.states, out.stats)
        return float((h.double() * wd).sum())

    grads = {"q": g.dq, "k": g.dk, "v": g.dv, "i_pre": g.d_ipre, "f_pre": g.d_fpre}
    report = {}
    for name, grad in grads.items():
        x = getattr(inp, name)
        gd = grad.double()
        if x.dtype == torch.bfloat16:  # linear in q / k / v: any step is exact
            d = torch.randn(x.shape, device="cuda", generator=gen, dtype=torch.float32)
            xp = (x.float() + 0.5 * d).to(torch.bfloat16)
            xm = (x.float() - 0.5 * d).to(torch.bfloat16)
        else:
            u = torch.rand(x.shape, device="cuda", generator=gen) + 0.5
            d = torch.sign(grad) * u
            xp, xm = x + 2e-2 * d, x - 2e-2 * d
        delta = xp.double() - xm.double()
        fields = {f: getattr(inp, f) for f in ("q", "k", "v", "i_pre", "f_pre")}
        lp = loss(SequenceInputs(**{**fields, name: xp.contiguous()}))
        lm = loss(SequenceInputs(**{**fields, name: xm.contiguous()}))
        fd = lp - lm
        an = float((gd * delta).sum())
        report[name] = abs(fd - an) / max(abs(an), 1e-30)
    print(f"variant={variant} L={L} FD rel err", {k_: f"{e:.2e}" for k_, e in report.items()})
    assert all(e < 3e-2 for e in report.values()), report
