"""Stabiliser audit on the B200 kernels: the GPU counterpart of the
reference's stab::exp_guarded counters (core.cpp:145-166).

test_tiled.cpp:135-145 and acceptance criterion 4 (acceptance.cpp:158) run a
tiled forward + backward and assert checks > 0 and violations == 0. Here the
kernels note every stabilised exponent argument before they clamp it at 0
(gates K0, the fused / split forward gating, the fused / split backward
gating, the decode step); a violation is an argument above 2^-10 in log2
units (fp32 rounding of an exactly-zero argument stays ~1e-5, a stabiliser
off by one log-gate is ~1). A deliberately wrong m_comb / m schedule must be
counted -- the audit is what keeps the fminf(arg, 0) clamps from hiding a
stabiliser bug.
"""
import numpy as np
import pytest

from tests._util import make_case, to_dev


@pytest.fixture
def audit():
    from paper_2503_14376_b200 import stab

    stab.enable(True)
    stab.reset()
    yield stab
    stab.enable(False)


def _fwd_bwd(B, H, T, L, dqk, dhv, variant, seed, f_bias=0.0, gate_scale=1.0):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed, f_bias=f_bias, gate_scale=gate_scale)
    inp = to_dev(q, k, v, ip, fp)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    out = chunkwise_forward(inp, dims, Variant(variant))
    dh = torch.randn(B, H, T, dhv, device="cuda").to(torch.bfloat16)
    chunkwise_backward(inp, dims, Variant(variant), dh, out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    return inp, dims, out


@pytest.mark.gpu
@pytest.mark.parametrize("L", [64, 128, 256, 512])
@pytest.mark.parametrize("gate_scale", [1.0, 2.0])
def test_no_stabiliser_violations(audit, fwd_path, L, gate_scale):
    """test_tiled.cpp:135-145 (make_inputs(d, rng, 1.0, 2.0)) on every kernel
    path: fused / split forward, fused (L=128) / split backward."""
    _fwd_bwd(1, 2, 1024, L, 128, 256, 0, seed=56 + L, gate_scale=gate_scale)
    checks, viol, amax = audit.read()
    print(f"L={L} scale={gate_scale} checks={checks} violations={viol} max_arg={amax:.2e}")
    assert checks > 0
    assert viol == 0
    assert amax < 1e-3


@pytest.mark.gpu
def test_no_violations_at_the_7b_head_shape(audit):
    _fwd_bwd(1, 1, 8192, 128, 256, 512, 0, seed=7, f_bias=3.0)
    checks, viol, amax = audit.read()
    assert checks > 8192 * 64  # every causal pair of every chunk, twice (fwd + bwd)
    assert viol == 0 and amax < 1e-3


@pytest.mark.gpu
def test_decode_step_is_audited(audit):
    import torch

    from paper_2503_14376_b200 import Dims, MemoryState, Variant, run_recurrent

    q, k, v, ip, fp = make_case(2, 2, 16, 64, 64, seed=3)
    dims = Dims(T=16, L=1, d_qk=64, d_hv=64, n_head=2, n_batch=2)
    run_recurrent(to_dev(q, k, v, ip, fp), dims, Variant.Exp, MemoryState.zero(dims))
    torch.cuda.synchronize()
    checks, viol, _ = audit.read()
    assert checks == 2 * 2 * 16 * 2 and viol == 0  # recurrent.cpp:17-18, two guarded exps per step


@pytest.mark.gpu
def test_wrong_stabiliser_is_counted(audit):
    """A frozen forward under an m_comb lowered by 2 puts positive arguments
    into the intra-chunk gating and b_bar: the audit must count them (the
    clamped kernels alone would return finite, wrong values)."""
    from paper_2503_14376_b200 import SavedStats, Variant, chunkwise_forward_frozen

    inp, dims, out = _fwd_bwd(1, 2, 512, 128, 64, 64, 0, seed=11)
    audit.reset()
    chunkwise_forward_frozen(inp, dims, Variant.Exp, out.states, out.stats)
    c0, v0, a0 = audit.read()
    assert c0 > 0 and v0 == 0
    bad = SavedStats(out.stats.m_combine - 2.0, out.stats.h_denom)
    chunkwise_forward_frozen(inp, dims, Variant.Exp, out.states, bad)
    c1, v1, a1 = audit.read()
    assert v1 > 0
    assert a1 > 1.5  # natural-log units: the 2.0 shift shows up as the largest argument
