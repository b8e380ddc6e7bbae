"""Chunkwise forward from an initial state (tfla_chunkwise_forward_init): the
chunkwise analogue of RecurrentOptions::initial_state (recurrent.hpp:23-27).

* forward vs the f64 recurrent oracle run from the same initial state
  (run_recurrent == chunkwise forward, acceptance.cpp:55-98): h <= TOL_H,
  final C / n <= TOL_H, m to fp32 rounding;
* segment split: forward + backward over [prefix ++ seq] vs forward from the
  prefix's final state over seq (+ backward): outputs, final states and the
  gradients on seq agree (the initial state is a constant of the segment).
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_H, make_case, np_, rel, to_dev


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", [(1, 2, 512, 128, 256, 256), (1, 1, 256, 64, 128, 128), (2, 1, 512, 256, 128, 256)])
def test_forward_from_state_matches_recurrent_oracle(case, variant, fwd_path):
    import torch

    from paper_2503_14376_b200 import Dims, MemoryState, Variant, chunkwise_forward

    B, H, T, L, dqk, dhv = case
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=T + L + variant)
    rng = np.random.default_rng(3)
    C0 = (rng.standard_normal((B, H, dqk, dhv)) * 0.5).astype(np.float32).astype(np.float64)
    n0 = np.abs(rng.standard_normal((B, H, dqk))).astype(np.float32).astype(np.float64)
    m0 = rng.standard_normal((B, H)).astype(np.float32).astype(np.float64)
    f32 = lambda a: torch.from_numpy(a).to("cuda", torch.float32).contiguous()
    init = MemoryState(f32(C0), f32(n0), f32(m0))
    out = chunkwise_forward(to_dev(q, k, v, ip, fp), Dims(T, L, dqk, dhv, H, B), Variant(variant),
                            initial_state=init)
    torch.cuda.synchronize()
    ref = Oracle().recurrent(q, k, v, ip, fp, variant, C0, n0, m0)
    errs = {"h": rel(np_(out.h_tilde), ref["h"]), "C": rel(np_(out.C_final), ref["C"])}
    if variant == 0:
        errs["n"] = rel(np_(out.n_final), ref["n"])
        assert np.abs(np_(out.m_final) - ref["m"]).max() < 1e-4 * (1 + np.abs(ref["m"]).max())
        assert np.abs(np_(out.states.m)[:, :, 0] - m0).max() == 0.0
    print(case, variant, fwd_path, {k_: f"{e:.2e}" for k_, e in errs.items()})
    for n, e in errs.items():
        assert e < TOL_H, (n, e)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_segment_split_forward_backward(variant, fwd_path):
    import torch

    from paper_2503_14376_b200 import Dims, MemoryState, SequenceInputs, Variant, chunkwise_backward, chunkwise_forward

    B, H, T0, T1, L, dqk, dhv = 1, 2, 512, 1024, 128, 256, 512
    T = T0 + T1
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=99 + variant)
    inp = to_dev(q, k, v, ip, fp)
    dh = bf16_round(np.random.default_rng(5).standard_normal((B, H, T, dhv)))
    dh[:, :, :T0] = 0.0
    dh_t = torch.from_numpy(dh).to("cuda", torch.bfloat16)
    full = chunkwise_forward(inp, Dims(T, L, dqk, dhv, H, B), Variant(variant))
    gfull = chunkwise_backward(inp, Dims(T, L, dqk, dhv, H, B), Variant(variant), dh_t, full.states, full.stats,
                               full.saved_states)
    kb = T0 // L
    init = MemoryState(full.states.C[:, :, kb].contiguous(), full.states.n[:, :, kb].contiguous(),
                       full.states.m[:, :, kb].contiguous())
    sl = lambda t: t[:, :, T0:].contiguous()
    seg = SequenceInputs(sl(inp.q), sl(inp.k), sl(inp.v), sl(inp.i_pre), sl(inp.f_pre))
    d1 = Dims(T1, L, dqk, dhv, H, B)
    part = chunkwise_forward(seg, d1, Variant(variant), initial_state=init)
    gpart = chunkwise_backward(seg, d1, Variant(variant), sl(dh_t), part.states, part.stats, part.saved_states)
    torch.cuda.synchronize()
    assert rel(np_(part.h_tilde), np_(full.h_tilde)[:, :, T0:]) < 1e-2
    assert rel(np_(part.C_final), np_(full.C_final)) < 1e-2
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        e = rel(np_(getattr(gpart, n)), np_(getattr(gfull, n))[:, :, T0:])
        print(variant, fwd_path, n, f"{e:.2e}")
        assert e < TOL_H, (n, e)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_initial_state_gradient_is_the_boundary_state_gradient(variant):
    """Stateful training across segments: the state pass of the second segment
    (forward from the first segment's final state) returns d_c[0] = dL/dC_0,
    which equals the full sequence's d_c at the segment boundary
    (backward_state_pass_head, chunkwise.cpp:196-237), and the chunk-sum
    partials d_g match there too."""
    import torch

    from paper_2503_14376_b200 import (Dims, MemoryState, SequenceInputs, Variant, backward_state_pass,
                                       chunkwise_forward)

    B, H, T0, T1, L, dqk, dhv = 1, 2, 512, 512, 128, 128, 256
    T = T0 + T1
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=123 + variant, f_bias=2.0)
    inp = to_dev(q, k, v, ip, fp)
    dh_t = torch.from_numpy(bf16_round(np.random.default_rng(6).standard_normal((B, H, T, dhv)))).to(
        "cuda", torch.bfloat16)
    dims = Dims(T, L, dqk, dhv, H, B)
    full = chunkwise_forward(inp, dims, Variant(variant))
    sp_full = backward_state_pass(inp, dims, Variant(variant), dh_t, full.states, full.stats, full.saved_states)
    kb = T0 // L
    init = MemoryState(full.states.C[:, :, kb].contiguous(), full.states.n[:, :, kb].contiguous(),
                       full.states.m[:, :, kb].contiguous())
    sl = lambda t: t[:, :, T0:].contiguous()
    seg = SequenceInputs(sl(inp.q), sl(inp.k), sl(inp.v), sl(inp.i_pre), sl(inp.f_pre))
    d1 = Dims(T1, L, dqk, dhv, H, B)
    part = chunkwise_forward(seg, d1, Variant(variant), initial_state=init)
    sp_part = backward_state_pass(seg, d1, Variant(variant), sl(dh_t), part.states, part.stats, part.saved_states)
    torch.cuda.synchronize()
    assert rel(np_(sp_part.d_c[:, :, 0]), np_(sp_full.d_c[:, :, kb])) < 1e-2
    assert rel(np_(sp_part.d_c), np_(sp_full.d_c[:, :, kb:])) < 1e-2
    assert rel(np_(sp_part.d_g), np_(sp_full.d_g[:, :, kb:])) < 2e-2
