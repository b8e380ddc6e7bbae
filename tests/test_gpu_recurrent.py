"""Recurrent (decode) path: run_recurrent (recurrent.cpp:65-115) with an
initial state, on the B200 kernel vs the f64 oracle restatement (itself pinned
to the reference in tests/test_oracle.py).

Tolerance (fp32 state, bf16 q/k/v in, bf16 h out; max_rel as in
gradcheck.cpp:7-10): h <= 1e-2, C / n final <= 1e-4 relative, m exact to fp32.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from tests._util import make_case, np_, rel, to_dev


def _state(B, H, dqk, dhv, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((B, H, dqk, dhv)) * 0.3, np.abs(rng.standard_normal((B, H, dqk))),
            rng.standard_normal((B, H)))


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape", [(2, 2, 1, 64, 64), (1, 3, 17, 128, 192), (2, 1, 64, 256, 512)])
@pytest.mark.parametrize("with_init", [False, True])
def test_recurrent_matches_oracle(variant, shape, with_init):
    import torch

    from paper_2503_14376_b200 import Dims, MemoryState, Variant, run_recurrent

    B, H, T, dqk, dhv = shape
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=T + dqk + variant)
    C0 = n0 = m0 = None
    init = None
    if with_init:
        C0, n0, m0 = _state(B, H, dqk, dhv, 9)
        C0 = C0.astype(np.float32).astype(np.float64)
        n0 = n0.astype(np.float32).astype(np.float64)
        m0 = m0.astype(np.float32).astype(np.float64)
        f32 = lambda a: torch.from_numpy(a).to("cuda", torch.float32).contiguous()
        init = MemoryState(f32(C0), f32(n0), f32(m0))
    ref = Oracle().recurrent(q, k, v, ip, fp, variant, C0, n0, m0)
    tr = run_recurrent(to_dev(q, k, v, ip, fp), Dims(T=T, L=1, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B),
                       Variant(variant), init)
    torch.cuda.synchronize()
    errs = {"h": rel(np_(tr.h_tilde), ref["h"]), "C": rel(np_(tr.C_final), ref["C"])}
    if variant == 0:
        errs["n"] = rel(np_(tr.n_final), ref["n"])
        assert np.abs(np_(tr.m_final) - ref["m"]).max() < 1e-4 * (1 + np.abs(ref["m"]).max())
    print(shape, variant, with_init, {k_: f"{e:.2e}" for k_, e in errs.items()})
    assert errs["h"] < 1e-2
    assert errs["C"] < 1e-4
    assert errs.get("n", 0.0) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_prefill_then_decode(variant):
    """Stateful inference: chunkwise_forward's final state (prefill of the first
    T0 tokens) handed to the recurrent kernel continues the sequence exactly
    like one recurrent run over all tokens."""
    import torch

    from paper_2503_14376_b200 import Dims, MemoryState, SequenceInputs, Variant, chunkwise_forward, run_recurrent

    B, H, T0, T1, L, dqk, dhv = 1, 2, 512, 8, 128, 256, 256
    q, k, v, ip, fp = make_case(B, H, T0 + T1, dqk, dhv, seed=77 + variant)
    inp = to_dev(q, k, v, ip, fp)
    sl = lambda t, a, b: t[:, :, a:b].contiguous()
    pre = SequenceInputs(*(sl(t, 0, T0) for t in (inp.q, inp.k, inp.v, inp.i_pre, inp.f_pre)))
    dec = SequenceInputs(*(sl(t, T0, T0 + T1) for t in (inp.q, inp.k, inp.v, inp.i_pre, inp.f_pre)))
    out = chunkwise_forward(pre, Dims(T0, L, dqk, dhv, H, B), Variant(variant), all_states=False)
    st = MemoryState(out.C_final.contiguous(), out.n_final.contiguous(), out.m_final.contiguous())
    tr = run_recurrent(dec, Dims(T1, 1, dqk, dhv, H, B), Variant(variant), st)
    torch.cuda.synchronize()
    ref = Oracle().recurrent(q, k, v, ip, fp, variant)
    assert rel(np_(tr.h_tilde), ref["h"][:, :, T0:]) < 2e-2
    assert rel(np_(tr.C_final), ref["C"]) < 2e-2


@pytest.mark.gpu
@pytest.mark.parametrize("T", [1, 3])
def test_decode_multiwave_grid_reads_initial_n_m(T):
    """every column-slice CTA of a head must see the INITIAL n / m.
    At the 7B decode shape (B=8, NH=8, dqk=256, dhv=512: 512 CTAs, more than
    one wave) with a non-zero initial m and n, a slice that started after
    slice 0 wrote the final n / m back would compute wrong gates and h."""
    import torch

    from paper_2503_14376_b200 import Dims, MemoryState, Variant, run_recurrent

    B, H, dqk, dhv = 8, 8, 256, 512
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=77 + T)
    C0, n0, m0 = _state(B, H, dqk, dhv, 13)
    C0 = C0.astype(np.float32).astype(np.float64)
    n0 = n0.astype(np.float32).astype(np.float64)
    m0 = (3.0 + m0).astype(np.float32).astype(np.float64)  # far from the step's m'
    f32 = lambda a: torch.from_numpy(a).to("cuda", torch.float32).contiguous()
    ref = Oracle().recurrent(q, k, v, ip, fp, 0, C0, n0, m0)
    for rep in range(3):
        tr = run_recurrent(to_dev(q, k, v, ip, fp), Dims(T=T, L=1, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B),
                           Variant.Exp, MemoryState(f32(C0), f32(n0), f32(m0)))
        torch.cuda.synchronize()
        assert rel(np_(tr.h_tilde), ref["h"]) < 1e-2
        assert rel(np_(tr.C_final), ref["C"]) < 1e-4
        assert rel(np_(tr.n_final), ref["n"]) < 1e-4
        assert np.abs(np_(tr.m_final) - ref["m"]).max() < 1e-4 * (1 + np.abs(ref["m"]).max())
