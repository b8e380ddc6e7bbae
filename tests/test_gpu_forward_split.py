"""Split forward entry points vs the f64 oracle.

tfla_state_recurrence = detail::state_recurrence_head (detail_kernels.hpp:38-44)
and tfla_forward_parallel = detail::tfla_forward_head (tiled.hpp:36-44), each
over every head. Tolerances as tests/test_gpu_forward.py:
  h, C states                <= TOL_H (1e-2)
  m states / m_combine       abs <= 1e-4 * (1+|ref|)
  h_denom, n states          <= 1e-2
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from tests._util import TOL_H, make_case, np_, rel, to_dev

CASES = [
    # B, H, T, L, dqk, dhv
    (1, 2, 256, 64, 64, 64),
    (1, 2, 512, 128, 128, 128),
    (1, 1, 384, 128, 256, 128),
    (2, 1, 256, 128, 256, 256),
]


def _m_err(x, ref):
    return float((np.abs(np_(x) - ref) / (1 + np.abs(ref))).max())


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
@pytest.mark.parametrize("via_saved", [True, False])
def test_state_recurrence_then_parallel_matches_oracle(case, variant, f_bias, via_saved):
    import torch

    from paper_2503_14376_b200 import BlockConfig, Dims, Variant, state_recurrence, tfla_forward_parallel

    B, H, T, L, dqk, dhv = case
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=hash(case) % 1000 + 7 * variant, f_bias=f_bias)
    ref = Oracle().forward(q, k, v, ip, fp, L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    states, saved = state_recurrence(inp, dims, Variant(variant), all_states=True, keep_saved=via_saved)
    out = tfla_forward_parallel(inp, dims, BlockConfig.pick_default(dims), Variant(variant), states,
                                saved if via_saved else None)
    torch.cuda.synchronize()
    assert rel(np_(states.C), ref["C"]) < TOL_H
    assert rel(np_(states.n), ref["n"]) < 1e-2
    assert _m_err(states.m, ref["m"]) < 1e-4
    assert rel(np_(out.h_tilde), ref["h"]) < TOL_H
    assert rel(np_(out.stats.h_denom), ref["h_denom"]) < 1e-2
    assert _m_err(out.stats.m_combine, ref["m_comb"]) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_parallel_from_oracle_states(variant):
    """tfla_forward_parallel consumes the caller's states (here the oracle's,
    in fp32) exactly as tfla_forward_head consumes state_recurrence_head's."""
    import torch

    from paper_2503_14376_b200 import BlockConfig, ChunkStates, Dims, Variant, tfla_forward_parallel

    B, H, T, L, dqk, dhv = 1, 2, 512, 128, 128, 256
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=91 + variant, f_bias=1.0)
    ref = Oracle().forward(q, k, v, ip, fp, L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float32)
    states = ChunkStates(f32(ref["C"]), f32(ref["n"]), f32(ref["m"]))
    out = tfla_forward_parallel(to_dev(q, k, v, ip, fp), dims, BlockConfig.pick_default(dims), Variant(variant),
                                states)
    torch.cuda.synchronize()
    assert rel(np_(out.h_tilde), ref["h"]) < TOL_H
    assert rel(np_(out.stats.h_denom), ref["h_denom"]) < 1e-2
    assert _m_err(out.stats.m_combine, ref["m_comb"]) < 1e-4


@pytest.mark.gpu
def test_split_forward_argument_errors():
    import torch

    from paper_2503_14376_b200 import (ChunkStates, Dims, ParameterError, Variant, state_recurrence,
                                       tfla_forward_parallel)

    q, k, v, ip, fp = make_case(1, 1, 256, 64, 64, seed=5)
    dims = Dims(T=256, L=64, d_qk=64, d_hv=64)
    inp = to_dev(q, k, v, ip, fp)
    with pytest.raises(ParameterError):
        state_recurrence(inp, dims, Variant.Exp, all_states=False, keep_saved=False)
    states, _ = state_recurrence(inp, dims, Variant.Exp)
    with pytest.raises(ParameterError):
        tfla_forward_parallel(inp, dims, None, Variant.Exp, states)
    from paper_2503_14376_b200 import BlockConfig

    no_n = ChunkStates(states.C, None, None)
    with pytest.raises(ParameterError):  # mLSTMexp needs n and m
        tfla_forward_parallel(inp, dims, BlockConfig.pick_default(dims), Variant.Exp, no_n)
    torch.cuda.synchronize()
