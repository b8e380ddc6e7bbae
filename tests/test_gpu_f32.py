"""fp32-operand forward (tfla_chunkwise_forward_f32, the reference's <float,
float> instantiation, chunkwise.cpp:183-194; BASELINE config 0 as worded) vs
the reference's golden fixtures and vs the f64 oracle on fp32 inputs that are
NOT bf16-rounded. fp32 operands and accumulation: max_rel <= 1e-4 on h, C, n
and h_denom (observed ~1e-6), m within 1e-5."""
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Oracle
from tests._util import np_, rel

FIX = sorted(p for p in (Path(__file__).parent / "golden").glob("cfg0_*.npz"))
TOL_F32 = 1e-4


def _inputs(q, k, v, ip, fp):
    import torch

    from paper_2503_14376_b200 import SequenceInputs

    f = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to("cuda")  # noqa: E731
    return SequenceInputs(f(q), f(k), f(v), f(ip), f(fp))


def _check(out, ref):
    errs = {"h": rel(np_(out.h_tilde), ref["h"]), "C": rel(np_(out.states.C), ref["C"]),
            "n": rel(np_(out.states.n), ref["n"]), "h_denom": rel(np_(out.stats.h_denom), ref["h_denom"])}
    m_err = float(np.abs(np_(out.states.m) - ref["m"]).max())
    print({k: f"{e:.2e}" for k, e in errs.items()}, "m", m_err)
    assert m_err < 1e-5
    for n, e in errs.items():
        assert e < TOL_F32, (n, e)


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIX, ids=[p.stem for p in FIX])
def test_f32_forward_matches_reference_golden(path):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward_f32
    from tests.golden.make_golden import load

    z = load(path)
    B, H, T, L, dqk, dhv, variant = (int(x) for x in z["dims"])
    out = chunkwise_forward_f32(_inputs(z["q"], z["k"], z["v"], z["i_pre"], z["f_pre"]),
                                Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), Variant(variant))
    torch.cuda.synchronize()
    _check(out, z)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 2, 256, 64, 64, 64), (2, 1, 384, 64, 128, 128), (1, 1, 256, 128, 64, 192)])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("f_bias", [0.0, 3.0])
def test_f32_forward_matches_oracle_unrounded(shape, variant, f_bias):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward_f32

    B, H, T, L, dqk, dhv = shape
    rng = np.random.default_rng(sum(shape) + variant)
    q, k = (rng.standard_normal((B, H, T, dqk)).astype(np.float32) for _ in range(2))
    v = rng.standard_normal((B, H, T, dhv)).astype(np.float32)
    ip = rng.standard_normal((B, H, T)).astype(np.float32)
    fp = (rng.standard_normal((B, H, T)) + f_bias).astype(np.float32)
    f64 = lambda a: a.astype(np.float64)  # noqa: E731
    ref = Oracle().forward(f64(q), f64(k), f64(v), f64(ip), f64(fp), L, variant)
    out = chunkwise_forward_f32(_inputs(q, k, v, ip, fp), Dims(T, L, dqk, dhv, H, B), Variant(variant))
    torch.cuda.synchronize()
    _check(out, {"h": ref["h"], "C": ref["C"], "n": ref["n"], "h_denom": ref["h_denom"], "m": ref["m"]})


@pytest.mark.gpu
def test_f32_forward_rejects_unsupported_geometry():
    import torch

    from paper_2503_14376_b200 import Dims, GeometryError, Variant, chunkwise_forward_f32

    B, H, T, L, dqk, dhv = 1, 1, 256, 128, 128, 64   # L * d_qk = 16384 > 8192
    z = lambda *s: torch.zeros(*s, device="cuda")  # noqa: E731
    from paper_2503_14376_b200 import SequenceInputs
    inp = SequenceInputs(z(B, H, T, dqk), z(B, H, T, dqk), z(B, H, T, dhv), z(B, H, T), z(B, H, T))
    with pytest.raises(GeometryError):
        chunkwise_forward_f32(inp, Dims(T, L, dqk, dhv, H, B), Variant.Exp)
