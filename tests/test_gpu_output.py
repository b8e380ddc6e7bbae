"""Output epilogue (eq. 5): sigmoid(o) * rms_norm(h_tilde; gamma, eps)
on the B200 kernel vs the f64 oracle restatement (pinned to the reference's
rms_norm, transfer.cpp:8-18, in tests/test_oracle.py). bf16 in / out:
max_rel <= 1e-2."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_H, np_, rel


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(2, 3, 17, 64), (1, 8, 128, 512), (1, 2, 4, 1024)])
@pytest.mark.parametrize("eps", [0.0, 1e-6])
def test_output_norm_gate_matches_oracle(shape, eps):
    import torch

    from paper_2503_14376_b200 import output_norm_gate

    B, H, T, d = shape
    rng = np.random.default_rng(sum(shape))
    x = bf16_round(rng.standard_normal(shape) * 0.3)
    x[0, 0, 0] = 0.0
    o = bf16_round(rng.standard_normal(shape))
    gamma = rng.standard_normal((H, d)).astype(np.float32).astype(np.float64)
    ref = Oracle().output_norm_gate(x, o, gamma, eps)
    bf = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16).contiguous()
    h = output_norm_gate(bf(x), bf(o), torch.from_numpy(gamma).to("cuda", torch.float32).contiguous(), eps)
    torch.cuda.synchronize()
    assert rel(np_(h), ref) < 1e-2
    assert float(h[0, 0, 0].float().abs().max()) == 0.0


@pytest.mark.gpu
def test_gate_softcap_matches_reference_formula():
    """apply_gate_softcap (gates.cpp:61-67) then the forward equals the oracle
    forward on capped pre-activations."""
    import torch

    from paper_2503_14376_b200 import Dims, Variant, apply_gate_softcap, chunkwise_forward
    from tests._util import make_case, to_dev

    B, H, T, L, d = 1, 2, 256, 64, 64
    q, k, v, ip, fp = make_case(B, H, T, d, d, seed=5, gate_scale=8.0)
    cap = 3.0
    capped = apply_gate_softcap(to_dev(q, k, v, ip, fp), cap)
    torch.cuda.synchronize()
    ic, fc = (cap * np.tanh(x / cap) for x in (ip, fp))
    assert np.abs(np_(capped.i_pre) - ic).max() < 1e-6 * cap
    assert np.abs(np_(capped.f_pre) - fc).max() < 1e-6 * cap
    out = chunkwise_forward(capped, Dims(T, L, d, d, H, B), Variant.Exp)
    ref = Oracle().forward(q, k, v, np_(capped.i_pre), np_(capped.f_pre), L, 0)
    assert rel(np_(out.h_tilde), ref["h"]) < TOL_H
    with pytest.raises(Exception):
        apply_gate_softcap(capped, 0.0)
