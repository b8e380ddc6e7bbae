"""The reference's known-answer tests for the step / sequence semantics
(test_recurrent.cpp:25-175), run on the B200 kernels: the recurrent decode
kernel for the single-step cases and both the decode kernel and the chunkwise
forward (K12 / K1+K2) for the sequence cases. The 4-wide vectors of the
reference are embedded in d_qk = d_hv = 64 (zero padded; q = k = 4 e1 keeps
k.q / sqrt(d_qk) = 2 as in the reference's q = k = 2 e1 at d_qk = 4).
Tolerances: results the reference checks to 1e-12 are exact up to the bf16
output rounding here (h is bf16: 2^-8 relative)."""
import numpy as np
import pytest

D = 64


def _inputs(T, q, k, v, ip, fp, B=1, H=1):
    import torch

    from paper_2503_14376_b200 import SequenceInputs

    bf = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float32)).reshape(B, H, T, -1).to("cuda", torch.bfloat16)
    f32 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float32)).reshape(B, H, T).to("cuda")
    return SequenceInputs(bf(q), bf(k), bf(v), f32(ip), f32(fp))


def _pad(vec, n=D):
    out = np.zeros(n)
    out[: len(vec)] = vec
    return out


def _run(inp, T, variant, L=None, init=None):
    from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward, run_recurrent

    if L is None:
        return run_recurrent(inp, Dims(T=T, L=1, d_qk=D, d_hv=D), Variant(variant), init)
    return chunkwise_forward(inp, Dims(T=T, L=L, d_qk=D, d_hv=D), Variant(variant), initial_state=init)


def _np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


@pytest.mark.gpu
def test_step_exp_saturated_gates_reproduce_v():
    """test_recurrent.cpp:25-35: i = 0, f = 1e3 -> m = 0 and h = v."""
    v = _pad([0.3, -1.2, 0.8])
    tr = _run(_inputs(1, _pad([4.0]), _pad([4.0]), v, [0.0], [1e3]), 1, 0)
    assert float(tr.m_final.item()) == 0.0
    assert np.allclose(_np(tr.h_tilde).ravel()[:3], v[:3], rtol=2 ** -8, atol=0)


@pytest.mark.gpu
def test_step_exp_max_state_lets_tiny_gates_pass():
    """test_recurrent.cpp:37-47: i = f = -1e3 -> m = -1e3 and C = k v^T."""
    tr = _run(_inputs(1, _pad([1.0]), _pad([1.0]), _pad([2.0, -1.0]), [-1e3], [-1e3]), 1, 0)
    assert abs(float(tr.m_final.item()) + 1e3) < 1e-3
    C = _np(tr.C_final)[0, 0]
    assert abs(C[0, 0] - 2.0) < 1e-6 and abs(C[0, 1] + 1.0) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_zero_value_and_state_give_zero_output(variant):
    """test_recurrent.cpp:49-55."""
    q = _pad([1, 1, 1, 1])
    k = _pad([1, 0, 1, 0])
    tr = _run(_inputs(1, q, k, np.zeros(D), [0.3], [0.1]), 1, variant)
    assert not _np(tr.h_tilde).any()


@pytest.mark.gpu
def test_step_sig_saturated_gates_give_half_v():
    """test_recurrent.cpp:57-65: i = 1e3 (sigma 1), f = -1e3, q.k/sqrt(d) = 1/2 -> h = v / 2
    (q = k = e1 scaled so k.q / sqrt(d_qk) = 1/8 * 4 = 1/2)."""
    v = _pad([1.0, 2.0, -3.0])
    tr = _run(_inputs(1, _pad([2.0]), _pad([2.0]), v, [1e3], [-1e3]), 1, 1)
    assert np.allclose(_np(tr.h_tilde).ravel()[:3], v[:3] / 2, rtol=2 ** -8, atol=0)


def _random(T, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    q, k = rng.standard_normal((T, D)) * scale, rng.standard_normal((T, D)) * scale
    v = rng.standard_normal((T, D))
    return q, k, v, rng.standard_normal(T), rng.standard_normal(T)


@pytest.mark.gpu
@pytest.mark.parametrize("L", [None, 64, 128])
def test_sig_blocked_input_stays_zero(L):
    """test_recurrent.cpp:67-74: sigma(i = -1e3) = 0 -> h = 0 (recurrent and chunkwise)."""
    T = 256
    q, k, v, _, fp = _random(T, 3)
    tr = _run(_inputs(T, q, k, v, np.full(T, -1e3), fp), T, 1, L)
    h = tr.h_tilde
    assert float(h.float().abs().max()) < 1e-30


@pytest.mark.gpu
@pytest.mark.parametrize("L", [None, 64, 128])
def test_exp_suppressed_input_stays_near_zero(L):
    """test_recurrent.cpp:94-102: i = -1e4, f = 0 -> |h| < 1e-6."""
    T = 256
    q, k, v, _, _ = _random(T, 4)
    tr = _run(_inputs(T, q, k, v, np.full(T, -1e4), np.zeros(T)), T, 0, L)
    assert float(tr.h_tilde.float().abs().max()) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("L", [None, 64, 128])
def test_sig_reduces_to_decayed_linear_attention(L):
    """test_recurrent.cpp:145-166: sigma(i) = 1, sigma(f) = gamma -> C_T = sum gamma^(T-1-t) k v^T."""
    gamma, T = 0.9, 256
    q, k, v, _, _ = _random(T, 12)
    inp = _inputs(T, q, k, v, np.full(T, 1e4), np.full(T, np.log(gamma / (1 - gamma))))
    out = _run(inp, T, 1, L)
    kb, vb = _np(inp.k)[0, 0], _np(inp.v)[0, 0]  # the bf16 values the kernels saw
    w = gamma ** (T - 1 - np.arange(T))
    expect = (kb * w[:, None]).T @ vb
    got = _np(out.C_final if L is None else out.C_final)[0, 0]
    assert np.abs(got - expect).max() / np.abs(expect).max() < (1e-5 if L is None else 1e-2)


@pytest.mark.gpu
@pytest.mark.parametrize("L", [None, 64])
def test_max_state_offset_cancels(L):
    """test_recurrent.cpp:127-143: starting from m_0 = -5 (zero C, n) gives the
    same outputs as m_0 = 0 (recurrent and chunkwise with an initial state)."""
    import torch

    from paper_2503_14376_b200 import Dims, MemoryState

    T = 128
    q, k, v, ip, fp = _random(T, 31)
    inp = _inputs(T, q, k, v, ip, fp)
    base = _run(inp, T, 0, L)
    shifted = MemoryState.zero(Dims(T=T, L=L or 1, d_qk=D, d_hv=D), "cuda")
    shifted.m.fill_(-5.0)
    moved = _run(inp, T, 0, L, init=shifted)
    torch.cuda.synchronize()
    a, b = _np(base.h_tilde), _np(moved.h_tilde)
    assert np.abs(a - b).max() <= 2 ** -7 * np.abs(a).max()


@pytest.mark.gpu
@pytest.mark.parametrize("L", [None, 64, 128])
def test_q_zero_gives_zero_output(L):
    """test_recurrent.cpp:168-175: q = 0 -> h = 0 exactly through the clamp."""
    T = 256
    _, k, v, ip, fp = _random(T, 8)
    tr = _run(_inputs(T, np.zeros((T, D)), k, v, ip, fp), T, 0, L)
    assert not _np(tr.h_tilde).any()


@pytest.mark.gpu
@pytest.mark.parametrize("where", ["q", "k", "v", "i_pre", "f_pre"])
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), float("-inf")])
def test_check_finite_flags_non_finite_inputs(where, bad):
    """SequenceInputs::validate's all_finite (core.cpp:106-117) -> NumericError,
    as the opt-in device pass tfla_check_finite; clean inputs pass."""
    import torch

    from paper_2503_14376_b200 import Dims, NumericError

    T = 193  # the gate buffers (772 B) end in a 4-byte tail past the last 16-byte word
    q, k, v, ip, fp = _random(T, 5)
    inp = _inputs(T, q, k, v, ip, fp, H=1)
    dims = Dims(T=T, L=1, d_qk=D, d_hv=D)
    inp.check_finite(dims)
    t = getattr(inp, where)
    t.view(-1)[t.numel() - 1] = bad  # last element: exercises the tail of the 16-byte sweep
    with pytest.raises(NumericError):
        inp.check_finite(dims)
    t.view(-1)[t.numel() - 1] = 0.0
    t.view(-1)[7] = bad
    with pytest.raises(NumericError):
        inp.check_finite(dims)
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("L", [64, 128, 1024])
def test_chunkwise_gates_match_oracle(variant, L):
    """tfla_chunkwise_gates (gates.cpp:20-59, f64 on the device) against the f64
    oracle (pinned to the reference's golden gates): same math, scan order only."""
    import torch

    from oracle.oracle import Oracle
    from paper_2503_14376_b200 import Dims, Variant, chunkwise_gates

    B, H, T = 2, 3, 2048
    rng = np.random.default_rng(L + variant)
    ip = (2 * rng.standard_normal((B, H, T))).astype(np.float32)
    fp = (2 * rng.standard_normal((B, H, T)) + 1).astype(np.float32)
    fp[0, 0, :64] = 1e3  # saturated forget gates: g = b = a = 0 (test_gates.cpp:64-72)
    out = chunkwise_gates(torch.from_numpy(fp).cuda(), torch.from_numpy(ip).cuda(), Dims(T=T, L=L, d_qk=64, d_hv=64,
                          n_head=H, n_batch=B), Variant(variant))
    torch.cuda.synchronize()
    orc = Oracle()
    for b in range(B):
        for h in range(H):
            g, bc, a = orc.gates(fp[b, h].astype(np.float64), ip[b, h].astype(np.float64), L, variant)
            assert np.allclose(out.g_sum[b, h].cpu().numpy(), g, rtol=1e-12, atol=1e-11)
            assert np.allclose(out.b_cum[b, h].cpu().numpy(), bc, rtol=1e-12, atol=1e-11)
            assert np.allclose(out.a_tail[b, h].cpu().numpy(), a, rtol=1e-12, atol=1e-11)
