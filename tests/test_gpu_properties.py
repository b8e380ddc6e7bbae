"""Size-independent properties at the BASELINE shapes (S=8192, dqk=256,
dhv=512), where the f64 oracle is too slow to check every head:
  - (b,h) slice independence, bit-exact (test_tiled.cpp:223-262)
  - zero upstream gradient -> exactly zero gradients (test_chunkwise.cpp:85-99)
  - chunk-size invariance L = 128 / 256 / 512 within the bf16 tolerance
  - block-config invariance of tfla_forward (output column tile 64 vs 128)
  - one full-size head pair checked against the f64 oracle
  - causality: poisoned future values leave earlier rows bit-exact
    (test_tiled.cpp:114-133); ascending maxima (:101-112); the denominator
    clamp (test_chunkwise.cpp:168-175); recurrent == chunkwise == parallel on
    the GPU kernels (test_chunkwise.cpp:27-44, acceptance criterion 1)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_H, make_case, np_, rel, to_dev


def _run(inp, dims, variant, dh=None, blocks=None):
    import torch

    from paper_2503_14376_b200 import Variant, chunkwise_backward, chunkwise_forward, tfla_forward

    out = (tfla_forward(inp, dims, blocks, Variant(variant), all_states=False) if blocks
           else chunkwise_forward(inp, dims, Variant(variant), all_states=False))
    g = None
    if dh is not None:
        g = chunkwise_backward(inp, dims, Variant(variant), dh, out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    return out, g


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_slice_independence_bitexact(variant, fwd_path):
    import torch

    from paper_2503_14376_b200 import Dims, SequenceInputs

    B, H, T, L, dqk, dhv = 2, 2, 1024, 128, 256, 512
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=3 + variant)
    dh = torch.from_numpy(bf16_round(np.random.default_rng(4).standard_normal((B, H, T, dhv)))).to("cuda", torch.bfloat16)
    inp = to_dev(q, k, v, ip, fp)
    full, gfull = _run(inp, Dims(T, L, dqk, dhv, H, B), variant, dh)
    for b in range(B):
        for h in range(H):
            sl = lambda t: t[b:b + 1, h:h + 1].contiguous()
            one = SequenceInputs(sl(inp.q), sl(inp.k), sl(inp.v), sl(inp.i_pre), sl(inp.f_pre))
            o, g = _run(one, Dims(T, L, dqk, dhv, 1, 1), variant, sl(dh))
            assert torch.equal(o.h_tilde[0, 0], full.h_tilde[b, h])
            for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
                assert torch.equal(getattr(g, n)[0, 0], getattr(gfull, n)[b, h]), n


@pytest.mark.gpu
def test_zero_dh_gives_zero_grads():
    import torch

    from paper_2503_14376_b200 import Dims

    B, H, T, L, dqk, dhv = 1, 2, 8192, 128, 256, 512
    inp = to_dev(*make_case(B, H, T, dqk, dhv, seed=8))
    for variant in (0, 1):
        _, g = _run(inp, Dims(T, L, dqk, dhv, H, B), variant,
                    torch.zeros(B, H, T, dhv, device="cuda", dtype=torch.bfloat16))
        for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
            assert float(getattr(g, n).abs().max()) == 0.0, n


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_chunk_size_invariance_full_shape(variant):
    import torch

    from paper_2503_14376_b200 import Dims

    B, H, T, dqk, dhv = 1, 2, 8192, 256, 512
    inp = to_dev(*make_case(B, H, T, dqk, dhv, seed=21 + variant))
    dh = torch.from_numpy(bf16_round(np.random.default_rng(22).standard_normal((B, H, T, dhv)))).to("cuda", torch.bfloat16)
    ref_o, ref_g = _run(inp, Dims(T, 128, dqk, dhv, H, B), variant, dh)
    for L in (256, 512):
        o, g = _run(inp, Dims(T, L, dqk, dhv, H, B), variant, dh)
        assert rel(np_(o.h_tilde), np_(ref_o.h_tilde)) < 2e-2
        for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
            assert rel(np_(getattr(g, n)), np_(getattr(ref_g, n))) < 4e-2, (L, n)


@pytest.mark.gpu
def test_block_config_invariance():
    from paper_2503_14376_b200 import BlockConfig, Dims

    B, H, T, L, dqk, dhv = 1, 2, 2048, 256, 256, 512
    inp = to_dev(*make_case(B, H, T, dqk, dhv, seed=31))
    dims = Dims(T, L, dqk, dhv, H, B)
    a, _ = _run(inp, dims, 0, blocks=BlockConfig(32, 8, 16, 64))
    b, _ = _run(inp, dims, 0, blocks=BlockConfig(32, 8, 16, 128))
    c, _ = _run(inp, dims, 0)
    assert rel(np_(a.h_tilde), np_(c.h_tilde)) < 1e-2
    assert rel(np_(b.h_tilde), np_(c.h_tilde)) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_full_shape_heads_vs_oracle(variant, fwd_path):
    """BASELINE configs[1] head shape (S=8192, dqk=256, dhv=512, L=128), two
    heads, forward and all gradients against the f64 oracle."""
    import torch

    from paper_2503_14376_b200 import Dims

    B, H, T, L, dqk, dhv = 1, 2, 8192, 128, 256, 512
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=41 + variant)
    dh = bf16_round(np.random.default_rng(42).standard_normal((B, H, T, dhv)))
    o, g = _run(to_dev(q, k, v, ip, fp), Dims(T, L, dqk, dhv, H, B), variant,
                torch.from_numpy(dh).to("cuda", torch.bfloat16))
    orc = Oracle()
    f = orc.forward(q, k, v, ip, fp, L, variant)
    rg = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
    errs = {"h": rel(np_(o.h_tilde), f["h"]), "C_final": rel(np_(o.C_final), f["C"][:, :, -1])}
    errs.update({n: rel(np_(getattr(g, n)), rg[n]) for n in ("dq", "dk", "dv", "d_fpre", "d_ipre")})
    print("full shape", variant, {k_: f"{e:.2e}" for k_, e in errs.items()})
    for n, e in errs.items():
        assert e < TOL_GRAD, (n, e)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_poisoned_future_values_leave_earlier_rows_bitexact(variant, fwd_path):
    """test_tiled.cpp:114-133: corrupting v at positions >= t0 (mid-chunk) must
    not change any earlier row: masked (j > i) score entries are exact zeros in
    the tensor-core accumulation, so rows < t0 are bit-identical."""
    import torch

    from paper_2503_14376_b200 import Dims

    B, H, T, L, dqk, dhv = 1, 2, 1024, 128, 256, 256
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=55 + variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    t0 = 3 * L + 40
    base, _ = _run(to_dev(q, k, v, ip, fp), dims, variant)
    vp = v.copy()
    vp[:, :, t0:] += 100.0
    pois, _ = _run(to_dev(q, k, vp, ip, fp), dims, variant)
    assert torch.equal(base.h_tilde[:, :, :t0], pois.h_tilde[:, :, :t0])
    assert torch.equal(base.stats.h_denom[:, :, :t0], pois.stats.h_denom[:, :, :t0])
    assert not torch.equal(base.h_tilde[:, :, t0:], pois.h_tilde[:, :, t0:])


@pytest.mark.gpu
def test_ascending_maxima_match_oracle(fwd_path):
    """test_tiled.cpp:101-112: strictly increasing input gates move the max
    state in every chunk (f = 2 keeps the memory); still within tolerance."""
    B, H, T, L, dqk, dhv = 1, 1, 512, 128, 128, 128
    q, k, v, _, _ = make_case(B, H, T, dqk, dhv, seed=54)
    ip = (-8.0 + 0.5 * np.arange(T)).astype(np.float32).astype(np.float64).reshape(B, H, T)
    fp = np.full((B, H, T), 2.0)
    ref = Oracle().forward(q, k, v, ip, fp, L, 0)
    from paper_2503_14376_b200 import Dims

    out, _ = _run(to_dev(q, k, v, ip, fp), Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), 0)
    assert rel(np_(out.h_tilde), ref["h"]) < TOL_H
    assert np.abs(np_(out.stats.m_combine) - ref["m_comb"]).max() < 1e-4 * (1 + np.abs(ref["m_comb"]).max())


@pytest.mark.gpu
def test_denominator_clamp(fwd_path):
    """test_chunkwise.cpp:168-175: h_denom >= exp(-m_comb) row by row (mLSTMexp)."""
    B, H, T, L, dqk, dhv = 2, 2, 512, 128, 256, 256
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=77, f_bias=1.0)
    from paper_2503_14376_b200 import Dims

    out, _ = _run(to_dev(q, k, v, ip, fp), Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), 0)
    den, mc = np_(out.stats.h_denom), np_(out.stats.m_combine)
    assert (den >= np.exp(-mc) * (1 - 1e-6)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_formulations_agree_on_gpu(variant):
    """test_chunkwise.cpp:27-44 / acceptance.cpp criterion 1 on the GPU kernels:
    recurrent decode (fp32 state, one step at a time) == chunkwise L = 64 ==
    chunkwise L = T (one chunk, the parallel formulation) within bf16 tolerance."""
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward, run_recurrent

    B, H, T, dqk, dhv = 1, 2, 512, 128, 128
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=81 + variant)
    inp = to_dev(q, k, v, ip, fp)
    rec = run_recurrent(inp, Dims(T=T, L=1, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), Variant(variant))
    c64 = chunkwise_forward(inp, Dims(T=T, L=64, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), Variant(variant))
    par = chunkwise_forward(inp, Dims(T=T, L=T, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), Variant(variant))
    torch.cuda.synchronize()
    r = np_(rec.h_tilde)
    assert rel(np_(c64.h_tilde), r) < 2e-2
    assert rel(np_(par.h_tilde), r) < 2e-2
    assert rel(np_(c64.C_final), np_(rec.C_final)) < 2e-2
