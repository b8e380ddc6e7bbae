"""CPU: pin the C restatement (oracle/tfla_oracle.c) before trusting it.

1. against the golden fixtures the reference itself produced (tests/golden);
2. against the reference library built from its own sources (oracle/_ref),
   when that library is present;
3. the reference's known-answer gate tests (test_gates.cpp:44-85) and
   properties of test_chunkwise.cpp (chunk-size invariance, zero dH).
"""
import math
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Oracle, Reference, max_rel
from tests.golden.make_golden import load

GOLDEN = sorted((Path(__file__).parent / "golden").glob("*.npz"))


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_oracle_matches_reference_golden(orc, path):
    z = load(path)
    B, H, T, L, dqk, dhv, variant = (int(x) for x in z["dims"])
    f = orc.forward(z["q"], z["k"], z["v"], z["i_pre"], z["f_pre"], L, variant)
    for name in ("h", "C", "n", "m", "m_comb", "h_denom"):
        assert max_rel(f[name], z[name]) < 1e-6, name
    g = orc.backward(z["q"], z["k"], z["v"], z["i_pre"], z["f_pre"], z["dh"], f["C"], f["m"], f["m_comb"],
                     f["h_denom"], L, variant)
    for name in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert max_rel(g[name], z[name]) < 1e-6, name


# ---- reference known answers for the gates (test_gates.cpp:44-85)
def test_gates_known_answers(orc):
    l2 = -0.6931471805599453
    g, b, a = orc.gates(np.zeros(4), np.zeros(4), 4, 0)
    assert g[0] == pytest.approx(4 * l2, rel=1e-14)
    assert np.allclose(b, [(j + 1) * l2 for j in range(4)], rtol=1e-14)
    assert np.allclose(a[:3], [3 * l2, 2 * l2, 1 * l2], rtol=1e-14) and a[3] == 0.0
    g, b, a = orc.gates(np.full(4, 1e3), np.zeros(4), 4, 0)
    assert abs(g[0]) < 1e-12 and np.abs(b).max() < 1e-12 and np.abs(a).max() < 1e-12


def test_gates_invariants(orc):
    rng = np.random.default_rng(5)
    T, L = 64, 16
    f, i = rng.standard_normal(T) * 3, rng.standard_normal(T) * 3
    for variant in (0, 1):
        g, b, a = orc.gates(f, i, L, variant)
        for k in range(T // L):
            bk = b[k * L:(k + 1) * L]
            assert abs(bk[-1] - g[k]) < 1e-12
            assert (bk <= 0).all() and (np.diff(bk) <= 0).all()
            ib = i[k * L:(k + 1) * L] if variant == 0 else [
                min(x, 0) - math.log1p(math.exp(-abs(x))) for x in i[k * L:(k + 1) * L]]
            assert np.abs(a[k * L:(k + 1) * L] - (g[k] - bk + ib)).max() < 1e-10
            assert a[k * L + L - 1] == ib[-1]


def _case(B, H, T, dqk, dhv, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((B, H, T, dqk)), rng.standard_normal((B, H, T, dqk)),
            rng.standard_normal((B, H, T, dhv)), rng.standard_normal((B, H, T)), rng.standard_normal((B, H, T)))


def test_chunk_size_invariance(orc):
    """test_chunkwise.cpp:46-65 / acceptance criterion 3: outputs and
    gradients do not depend on L."""
    q, k, v, ip, fp = _case(1, 2, 128, 8, 12, 43)
    dh = np.random.default_rng(1).standard_normal((1, 2, 128, 12))
    for variant in (0, 1):
        ref_h = ref_g = None
        for L in (8, 16, 32, 64):
            f = orc.forward(q, k, v, ip, fp, L, variant)
            g = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
            if ref_h is None:
                ref_h, ref_g = f["h"], g
                continue
            assert np.abs(f["h"] - ref_h).max() < 1e-10
            for n in g:
                assert np.abs(g[n] - ref_g[n]).max() < 1e-9, n


def test_zero_dh_zero_grads(orc):
    q, k, v, ip, fp = _case(1, 1, 16, 4, 4, 3)
    for variant in (0, 1):
        f = orc.forward(q, k, v, ip, fp, 4, variant)
        g = orc.backward(q, k, v, ip, fp, np.zeros((1, 1, 16, 4)), f["C"], f["m"], f["m_comb"], f["h_denom"], 4,
                         variant)
        assert all(np.abs(x).max() == 0.0 for x in g.values())


def test_clamp_definition(orc):
    """test_chunkwise.cpp:168-175: h_denom >= exp(-m_combine)."""
    q, k, v, ip, fp = _case(1, 1, 64, 8, 8, 47)
    f = orc.forward(q, k, v, ip, fp, 16, 0)
    assert (f["h_denom"] >= np.exp(-f["m_comb"]) * (1 - 1e-15)).all()


# ---- live comparison with the reference library (when built here)
needs_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape", [(1, 2, 256, 64, 64, 64), (2, 2, 128, 32, 16, 24), (1, 1, 24, 1, 6, 6)])
def test_oracle_matches_live_reference(orc, variant, shape):
    B, H, T, L, dqk, dhv = shape
    ref = Reference()
    q, k, v, ip, fp = ref.make_inputs(B, H, T, dqk, dhv, seed=11)
    dh = ref.normals(12, 0, B * H * T * dhv).reshape(B, H, T, dhv)
    fo, fr = orc.forward(q, k, v, ip, fp, L, variant), ref.forward(q, k, v, ip, fp, L, variant)
    for n in fo:
        assert max_rel(fo[n], fr[n]) < 1e-12, n
    go = orc.backward(q, k, v, ip, fp, dh, fr["C"], fr["m"], fr["m_comb"], fr["h_denom"], L, variant)
    gr = ref.backward(q, k, v, ip, fp, dh, fr["C"], fr["n"], fr["m"], fr["m_comb"], fr["h_denom"], L, variant)
    for n in go:
        assert max_rel(go[n], gr[n]) < 1e-12, n


@needs_ref
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape,blocks", [((1, 2, 256, 64, 64, 64), (32, 8, 16, 32)),
                                          ((2, 1, 96, 32, 16, 24), (16, 8, 8, 8))])
def test_oracle_split_partials_match_live_reference(orc, variant, shape, blocks):
    """The oracle's split-entry-point partials against the reference's own
    tfla_backward_dq / _dk / _dv (tiled.cpp:391-779) and
    backward_state_pass_head (chunkwise.cpp:196-237)."""
    B, H, T, L, dqk, dhv = shape
    ref = Reference()
    q, k, v, ip, fp = ref.make_inputs(B, H, T, dqk, dhv, seed=21)
    dh = ref.normals(22, 0, B * H * T * dhv).reshape(B, H, T, dhv)
    fr = ref.forward(q, k, v, ip, fp, L, variant)
    go = orc.backward_parts(q, k, v, ip, fp, dh, fr["C"], fr["m"], fr["m_comb"], fr["h_denom"], L, variant)
    gr = ref.backward_split(q, k, v, ip, fp, dh, fr["C"], fr["n"], fr["m"], fr["m_comb"], fr["h_denom"], L,
                            variant, blocks)
    for n in gr:
        assert max_rel(go[n], gr[n]) < 1e-12, n
    # assembly identity: the oracle's full d_fpre / d_ipre use d_b_q + d_b_kv (tiled.cpp:803)
    full = ref.backward(q, k, v, ip, fp, dh, fr["C"], fr["n"], fr["m"], fr["m_comb"], fr["h_denom"], L, variant,
                        blocks=blocks)
    for n in ("d_fpre", "d_ipre"):
        assert max_rel(go[n], full[n]) < 1e-12, n


@needs_ref
def test_reference_equivalences_and_gradcheck():
    """Acceptance criteria 1-2 of the reference (acceptance.cpp:55-98) on the
    library built from its own sources: recurrent == parallel == chunkwise ==
    tiled, and the analytic backward matches central differences."""
    ref = Reference()
    q, k, v, ip, fp = ref.make_inputs(1, 2, 64, 16, 32, seed=1001)
    for variant in (0, 1):
        rec = ref.recurrent(q, k, v, ip, fp, variant)["h"]
        par = ref.parallel(q, k, v, ip, fp, variant)
        cw = ref.forward(q, k, v, ip, fp, 16, variant)["h"]
        tf = ref.forward(q, k, v, ip, fp, 16, variant, blocks=(8, 4, 16, 32))["h"]
        for x in (par, cw, tf):
            assert np.abs(x - rec).max() < 1e-8
    q, k, v, ip, fp = ref.make_inputs(1, 1, 16, 4, 4, seed=2002)
    w = ref.normals(7, 0, 64).reshape(1, 1, 16, 4)
    for variant in (0, 1):
        rep = ref.gradcheck(q, k, v, ip, fp, w, 4, variant)
        assert max(rep.values()) < 1e-5, rep


# ---- recurrent (decode) path: run_recurrent (recurrent.cpp:65-115)
@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_recurrent_matches_reference_golden(orc, path):
    """The step recurrence reproduces the reference's chunkwise outputs and
    final states (the reference's own equivalence, acceptance.cpp:55-98)."""
    z = load(path)
    variant = int(z["dims"][6])
    r = orc.recurrent(z["q"], z["k"], z["v"], z["i_pre"], z["f_pre"], variant)
    # (fixtures are stored in fp32: 1e-6 is their resolution)
    assert max_rel(r["h"], z["h"]) < 1e-6
    assert max_rel(r["C"], z["C"][:, :, -1]) < 1e-6
    if variant == 0:
        assert max_rel(r["n"], z["n"][:, :, -1]) < 1e-6
        assert np.abs(r["m"] - z["m"][:, :, -1]).max() < 1e-6


@needs_ref
@pytest.mark.parametrize("variant", [0, 1])
def test_recurrent_matches_live_reference(orc, variant):
    ref = Reference()
    q, k, v, ip, fp = ref.make_inputs(2, 2, 48, 16, 24, seed=31)
    a, b = orc.recurrent(q, k, v, ip, fp, variant), ref.recurrent(q, k, v, ip, fp, variant)
    for n, rn in (("h", "h"), ("C", "C_final"), ("n", "n_final"), ("m", "m_final")):
        assert max_rel(a[n], b[rn]) < 1e-12, n


@pytest.mark.parametrize("variant", [0, 1])
def test_recurrent_initial_state_split(orc, variant):
    """Carrying the final state into a second run (RecurrentOptions::initial_state,
    recurrent.hpp:23-27) equals one run over the concatenated sequence."""
    rng = np.random.default_rng(5)
    B, H, T, dqk, dhv, T1 = 1, 2, 40, 8, 12, 17
    q, k = rng.standard_normal((2, B, H, T, dqk))
    v = rng.standard_normal((B, H, T, dhv))
    ip, fp = rng.standard_normal((2, B, H, T))
    full = orc.recurrent(q, k, v, ip, fp, variant)
    s = lambda x, a, b: np.ascontiguousarray(x[:, :, a:b])
    one = orc.recurrent(s(q, 0, T1), s(k, 0, T1), s(v, 0, T1), s(ip, 0, T1), s(fp, 0, T1), variant)
    two = orc.recurrent(s(q, T1, T), s(k, T1, T), s(v, T1, T), s(ip, T1, T), s(fp, T1, T), variant,
                        one["C"], one["n"], one["m"])
    assert max_rel(np.concatenate([one["h"], two["h"]], axis=2), full["h"]) < 1e-12
    for n in ("C", "n", "m"):
        assert max_rel(two[n], full[n]) < 1e-12, n


# ---- output epilogue (eq. 5): sigmoid(o) * rms_norm(h_tilde)
def test_output_norm_gate_matches_reference_rms_norm(orc):
    rng = np.random.default_rng(4)
    B, H, T, d = 2, 3, 5, 16
    x = rng.standard_normal((B, H, T, d))
    x[0, 0, 0] = 0.0  # zero row: rms == 0 convention (eps = 0)
    o = rng.standard_normal((B, H, T, d))
    gamma = rng.standard_normal((H, d))
    for eps in (0.0, 1e-6):
        out = orc.output_norm_gate(x, o, gamma, eps)
        if Reference.available():
            ref = Reference()
            for h in range(H):
                y = ref.rms_norm(np.ascontiguousarray(x[:, h]), np.ascontiguousarray(gamma[h]), eps)
                exp = 1.0 / (1.0 + np.exp(-o[:, h])) * y
                assert np.abs(out[:, h] - exp).max() < 1e-12
        assert np.all(out[0, 0, 0] == 0.0) if eps == 0.0 else True
