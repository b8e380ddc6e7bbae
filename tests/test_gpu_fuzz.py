"""Randomised parity sweep: 48 seeded geometries (chunk sizes 64..512, d_qk up to
512 / d_hv up to 512, multiples of 64 incl. partial 128-tiles, 1..3 chunks per sequence, batch and head
counts 1..3, both variants, forget-gate biases and gate scales) through the
default library path, forward + backward against the f64 oracle. Tolerances as
test_gpu_forward / test_gpu_backward (h, C <= TOL_H; gradients <= TOL_GRAD)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_H, make_case, np_, rel, to_dev


def _configs(n=48, seed=2025):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        L = int(rng.choice([64, 128, 128, 256, 512]))
        T = L * int(rng.integers(1, 4))
        dqk = int(rng.choice([64, 128, 192, 256, 320, 384, 512]))
        dhv = int(rng.choice([64, 128, 192, 256, 384, 512]))
        B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        variant = int(rng.integers(0, 2))
        f_bias = float(rng.choice([-2.0, 0.0, 3.0]))
        gate_scale = float(rng.choice([0.5, 1.0, 3.0]))
        out.append((B, H, T, L, dqk, dhv, variant, f_bias, gate_scale))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", _configs(), ids=lambda c: "B{}H{}T{}L{}q{}v{}var{}f{}g{}".format(*c))
def test_random_geometry_matches_oracle(cfg):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    B, H, T, L, dqk, dhv, variant, f_bias, gate_scale = cfg
    seed = abs(hash(cfg)) % 10000
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=seed, f_bias=f_bias, gate_scale=gate_scale)
    dh = bf16_round(np.random.default_rng(seed + 1).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    f = orc.forward(q, k, v, ip, fp, L, variant)
    g = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    gd = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                            out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    assert rel(np_(out.h_tilde), f["h"]) < TOL_H
    assert rel(np_(out.states.C), f["C"]) < TOL_H
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rel(np_(getattr(gd, n)), g[n]) < TOL_GRAD, n
