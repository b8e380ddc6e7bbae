"""Large chunk sizes (BASELINE configs[2]: the L sweep up to 1024): the split
K1 + K2 forward and the three dQ / dK / dV kernels tile the intra-chunk
matmuls over 128-row / 128-column blocks of arbitrarily large chunks
(tiled.cpp:59-240). Parity against the f64 oracle with the tolerances of
test_gpu_forward / test_gpu_backward (H <= TOL_H, gradients <= TOL_GRAD)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_H, make_case, np_, rel, to_dev


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", [(1, 1, 2048, 1024, 64, 64), (1, 1, 1024, 512, 128, 128),
                                  (1, 1, 2048, 1024, 256, 512)])
def test_large_chunk_fwd_bwd_matches_oracle(case, variant):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    B, H, T, L, dqk, dhv = case
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=3 + variant, f_bias=1.0)
    dh = bf16_round(np.random.default_rng(4).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    f = orc.forward(q, k, v, ip, fp, L, variant)
    g = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    gg = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                            out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    assert rel(np_(out.h_tilde), f["h"]) < TOL_H
    assert rel(np_(out.states.C), f["C"]) < TOL_H
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rel(np_(getattr(gg, n)), g[n]) < TOL_GRAD, n


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", [(1, 1, 256, 128, 512, 512), (1, 1, 256, 128, 128, 4096), (1, 1, 384, 128, 256, 2048)])
def test_maximum_head_dims_match_oracle(case, variant, fwd_path):
    """The largest head dimensions the C ABI accepts (d_qk <= 512, d_hv <= 4096,
    capi.cpp validate_dims) through both forward paths and the backward."""
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    B, H, T, L, dqk, dhv = case
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=17 + variant)
    dh = bf16_round(np.random.default_rng(18).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    f = orc.forward(q, k, v, ip, fp, L, variant)
    g = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    gg = chunkwise_backward(inp, dims, Variant(variant), torch.from_numpy(dh).to("cuda", torch.bfloat16),
                            out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    assert rel(np_(out.h_tilde), f["h"]) < TOL_H
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rel(np_(getattr(gg, n)), g[n]) < TOL_GRAD, n
