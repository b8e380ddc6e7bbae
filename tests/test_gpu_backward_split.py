"""Split backward entry points vs the f64 oracle.

tfla_backward_dq / _dk / _dv (tiled.hpp:56-84 / tiled.cpp:391-779), the state
pass (backward_state_pass_head, chunkwise.cpp:196-237) and the gate assembly
(assemble_gate_grads_head, chunkwise.cpp:239-266). The oracle's partials are
pinned to the reference's own split entry points in
tests/test_oracle.py::test_oracle_split_partials_match_live_reference.

Tolerance (bf16 tensor-core operands, fp32 accumulation; max_rel = max|x-ref| /
max|ref|): every gradient and partial <= TOL_GRAD (1.5e-2), as test_gpu_backward. The
assembly fed the oracle's own partials in fp32 is checked at 1e-5.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, make_case, np_, rel, to_dev

CASES = [
    # B, H, T, L, dqk, dhv
    (1, 2, 256, 64, 64, 64),
    (1, 2, 512, 128, 128, 128),
    (1, 1, 384, 128, 256, 128),
    (1, 2, 384, 128, 256, 256),
]


def _setup(case, variant, f_bias):
    import torch

    from paper_2503_14376_b200 import BlockConfig, Dims, Variant, chunkwise_forward

    B, H, T, L, dqk, dhv = case
    seed = hash(case) % 1000 + 31 * variant
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=seed, f_bias=f_bias)
    dh = bf16_round(np.random.default_rng(seed + 1).standard_normal((B, H, T, dhv)))
    orc = Oracle()
    fwd = orc.forward(q, k, v, ip, fp, L, variant)
    ref = orc.backward_parts(q, k, v, ip, fp, dh, fwd["C"], fwd["m"], fwd["m_comb"], fwd["h_denom"], L, variant)
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(q, k, v, ip, fp)
    out = chunkwise_forward(inp, dims, Variant(variant))
    dh_t = torch.from_numpy(dh).to("cuda", torch.bfloat16)
    return dims, BlockConfig.pick_default(dims), inp, out, dh_t, ref


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
@pytest.mark.parametrize("from_fp32_states", [False, True])
def test_split_entry_points_match_oracle(case, variant, f_bias, from_fp32_states):
    import torch

    from paper_2503_14376_b200 import (Variant, assemble_gate_grads, backward_state_pass, tfla_backward_dk,
                                       tfla_backward_dq, tfla_backward_dv)

    dims, blocks, inp, out, dh, ref = _setup(case, variant, f_bias)
    saved = None if from_fp32_states else out.saved_states
    var = Variant(variant)
    rq = tfla_backward_dq(inp, dims, blocks, var, dh, out.states, out.stats, saved)
    rk = tfla_backward_dk(inp, dims, blocks, var, dh, out.states, out.stats, saved)
    dv = tfla_backward_dv(inp, dims, blocks, var, dh, out.states, out.stats, saved)
    sp = backward_state_pass(inp, dims, var, dh, out.states, out.stats, saved)
    dfp, dip = assemble_gate_grads(inp, dims, var, sp.d_g, rq.d_b_cum + rk.d_b_cum, rk.d_a_tail, rk.d_i_log)
    torch.cuda.synchronize()
    got = {"dq": rq.dq, "d_b_q": rq.d_b_cum, "dk": rk.dk, "d_a_tail": rk.d_a_tail, "d_b_kv": rk.d_b_cum,
           "d_i_log": rk.d_i_log, "dv": dv, "d_g": sp.d_g, "d_c": sp.d_c, "d_fpre": dfp, "d_ipre": dip}
    errs = {n: rel(np_(t), ref[n]) for n, t in got.items()}
    print(case, variant, f_bias, from_fp32_states, {k_: f"{e:.2e}" for k_, e in errs.items()})
    for n, e in errs.items():
        assert e < TOL_GRAD, (n, e)
    # TfLaDkResult's two column-sum partials are exact negatives (tiled.cpp:628-629)
    assert torch.equal(rk.d_b_cum, -rk.d_i_log)
    # d_c entry NC is the zero boundary (chunkwise.cpp:206)
    assert not sp.d_c[:, :, -1].any()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_assembly_of_oracle_partials(variant):
    """assemble_gate_grads on the oracle's partials (fp32) reproduces the
    oracle's d_fpre / d_ipre: isolates the assembly kernel."""
    import torch

    from paper_2503_14376_b200 import Variant, assemble_gate_grads

    dims, _, inp, _, _, ref = _setup((2, 2, 512, 128, 64, 64), variant, 1.0)
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float32)
    dfp, dip = assemble_gate_grads(inp, dims, Variant(variant), f32(ref["d_g"]), f32(ref["d_b_q"] + ref["d_b_kv"]),
                                   f32(ref["d_a_tail"]), f32(ref["d_i_log"]))
    torch.cuda.synchronize()
    assert rel(np_(dfp), ref["d_fpre"]) < 1e-5
    assert rel(np_(dip), ref["d_ipre"]) < 1e-5


@pytest.mark.gpu
def test_split_backward_requires_blocks():
    from paper_2503_14376_b200 import ParameterError, Variant, tfla_backward_dq

    dims, _, inp, out, dh, _ = _setup((1, 1, 256, 64, 64, 64), 0, 0.0)
    with pytest.raises(ParameterError):
        tfla_backward_dq(inp, dims, None, Variant.Exp, dh, out.states, out.stats)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_query_side_gate_partial_is_dh_dot_h(variant):
    """TfLaDqResult::d_b_cum is dL/db_i with the normaliser detached; every term
    of h_tilde_i (intra through D_ij, inter through b_bar_i) scales with
    exp(b_i), so the partial equals dh_i . h_tilde_i row by row -- an identity
    that checks the dQ kernel's row sums and q.(dH C^T) dots without the oracle."""
    import torch

    from paper_2503_14376_b200 import Variant, tfla_backward_dq

    dims, blocks, inp, out, dh, _ = _setup((1, 2, 512, 128, 128, 128), variant, 1.0)
    rq = tfla_backward_dq(inp, dims, blocks, Variant(variant), dh, out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    ident = (dh.float() * out.h_tilde.float()).sum(-1)
    err = (rq.d_b_cum - ident).abs().max().item() / ident.abs().max().item()
    assert err < TOL_GRAD, err


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", [(1, 2, 512, 128, 128, 128), (1, 1, 384, 64, 64, 128)])
def test_input_gate_gradient_is_v_dot_dv(variant, case):
    """The input gate enters only as a scale of token j's value contribution
    (e^{i_j} resp. sigma(i_j) on k_j v_j^T and on D_ij), so
    d_ipre_j = (v_j . dv_j) (mLSTMexp) resp. (v_j . dv_j) sigma(-i_j) (mLSTMsig):
    checks the key-side partials (d_a, column sums) and the assembly against
    the dV kernel, without the oracle."""
    import torch

    from paper_2503_14376_b200 import Variant, chunkwise_backward

    dims, _, inp, out, dh, _ = _setup(case, variant, 1.0)
    g = chunkwise_backward(inp, dims, Variant(variant), dh, out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    ident = (inp.v.float() * g.dv.float()).sum(-1)
    if variant == 1:
        ident = ident * torch.sigmoid(-inp.i_pre.double()).float()
    err = (g.d_ipre - ident).abs().max().item() / ident.abs().max().item()
    assert err < TOL_GRAD, err
