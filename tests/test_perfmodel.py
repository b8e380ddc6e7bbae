"""The cost model (paper_2503_14376_b200/perfmodel.py) against the reference's
own perfmodel.cpp built from its sources (oracle/_ref), plus the reference's
documented properties (perfmodel.hpp). CPU only."""
import math

import numpy as np
import pytest

from oracle.oracle import Reference
from paper_2503_14376_b200 import Dims, ParameterError, Variant
from paper_2503_14376_b200 import perfmodel as pm

needs_pm = pytest.mark.skipif(not (Reference.available() and Reference().has_perfmodel()),
                              reason="oracle/_ref without perfmodel.cpp")

POINTS = [
    # variant, B, H, T, L, dqk, dhv
    (0, 8, 8, 8192, 128, 256, 512),   # BASELINE 7B shape
    (1, 8, 8, 8192, 256, 256, 512),
    (0, 1, 8, 65536, 128, 256, 512),  # long context
    (1, 1, 2, 256, 64, 64, 64),       # oracle config
    (0, 2, 3, 96, 32, 16, 24),
]
PARAMS = [
    pm.PerfParams(),
    pm.PerfParams(f_causal=1.0, f_exp=3.0, f_log=2.0, f_sig=4.0, f_max=1.5, f_abs=0.5, f_mask=2.0,
                  bytes_qkv=4.0, bytes_if=4.0, bytes_cmn=2.0),
]
ACCELS = [pm.AcceleratorSpec("B200 measured", 1628.2e12, 6556.8e9), pm.PRESETS[2]]


def _ours(pt, prm, acc):
    v, B, H, T, L, dqk, dhv = pt
    d = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    var = Variant(v)
    out = []
    for simp in (False, True):
        out += [x for _, x in pm.flops_chunkwise(d, prm, var, simp).items]
    out += [x for _, x in pm.flops_parallel(d, prm, var).items]
    out += [x for _, x in pm.flops_recurrent(d, prm, var).items]
    for f in ("chunkwise", "parallel", "recurrent"):
        m = pm.memops(d, prm, var, f)
        out += [m.loaded, m.stored]
    pqk = dqk / dhv
    ai = pm.arithmetic_intensity(d, prm, L)
    cands = pm.chunk_size_candidates(16, 1024, T)
    out += [pm.chunkwise_flops_model(var, T, L, dqk, dhv, prm.f_causal),
            pm.chunkwise_bytes_model(var, T, L, dqk, dhv, prm),
            pm.flop_optimal_chunk_size(dhv, pqk, prm.f_causal),
            pm.runtime_optimal_chunk_size(dhv, pqk, prm.f_causal, prm.bytes_cmn, pm.accelerator_intensity(acc)),
            pm.theoretical_runtime(d, prm, var, acc, L, "sum"), pm.theoretical_runtime(d, prm, var, acc, L, "max"),
            ai, pm.accelerator_intensity(acc), pm.roofline(acc, ai),
            pm.flop_argmin_chunk_size(dhv, pqk, prm.f_causal, cands),
            pm.runtime_argmin_chunk_size(dhv, pqk, prm.f_causal, prm.bytes_cmn, acc, cands)]
    return np.array(out, dtype=np.float64)


@needs_pm
@pytest.mark.parametrize("pt", POINTS)
@pytest.mark.parametrize("pi", range(len(PARAMS)))
@pytest.mark.parametrize("ai", range(len(ACCELS)))
def test_perfmodel_matches_reference(pt, pi, ai):
    prm, acc = PARAMS[pi], ACCELS[ai]
    vec = [prm.f_causal, prm.f_exp, prm.f_log, prm.f_sig, prm.f_max, prm.f_abs, prm.f_mask,
           prm.bytes_qkv, prm.bytes_if, prm.bytes_cmn]
    ref = Reference().perfmodel(*pt, vec, acc.flops_per_s, acc.bytes_per_s)
    ours = _ours(pt, prm, acc)
    err = np.abs(ours - ref) / np.maximum(np.abs(ref), 1e-300)
    err[ref == 0] = np.abs(ours[ref == 0])
    assert err.max() < 1e-12, (int(err.argmax()), ours[err.argmax()], ref[err.argmax()])


def test_optimal_chunk_size_is_stationary_point():
    """flop_optimal_chunk_size is the stationary point of the sigmoid FLOP
    polynomial in L (perfmodel.hpp:62-72)."""
    dhv, pqk, fc = 512.0, 0.5, 0.5
    L0 = pm.flop_optimal_chunk_size(dhv, pqk, fc)
    f = lambda L: pm.chunkwise_flops_model(Variant.Sig, 8192.0, L, pqk * dhv, dhv, fc)
    h = 1e-3 * L0
    assert abs(f(L0 + h) - f(L0 - h)) / (2 * h) < 1e-6 * f(L0) / L0
    assert f(L0) < f(0.5 * L0) and f(L0) < f(2 * L0)


def test_validation_and_presets():
    with pytest.raises(ParameterError):
        pm.PerfParams(f_causal=0.4).validate()
    with pytest.raises(ParameterError):
        pm.PerfParams(bytes_qkv=3.0).validate()
    with pytest.raises(ParameterError):
        pm.chunk_size_candidates(0, 4, 16)
    assert pm.chunk_size_candidates(16, 1024, 8192) == [16, 32, 64, 128, 256, 512, 1024]
    assert pm.find_accelerator("B200 HGX").flops_per_s == 2250e12
    with pytest.raises(ParameterError):
        pm.find_accelerator("TPU")


def test_measured_b200_report():
    """bench.py's roofline reporter: the model on the measured B200 of this pool."""
    acc = pm.measured_b200()
    assert acc.flops_per_s > 1e15 and acc.bytes_per_s > 1e12
    d = Dims(T=8192, L=128, d_qk=256, d_hv=512, n_head=8, n_batch=8)
    r = pm.report(d, Variant.Exp, acc)
    assert math.isclose(r["fwd_model_ms_max"], 1e3 * pm.theoretical_runtime(d, pm.PerfParams(), Variant.Exp, acc,
                                                                             128, "max"))
    assert r["fwd_model_ms_sum"] >= r["fwd_model_ms_max"] > 0
