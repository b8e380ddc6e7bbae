"""Output epilogue (eq. 5): sigmoid(o) * rms_norm(h_tilde; gamma, eps)
on the B200 kernel vs the f64 oracle restatement (pinned to the reference's
rms_norm, transfer.cpp:8-18, in tests/test_oracle.py). bf16 in / out:
max_rel <= 1e-2."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import np_, rel


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
