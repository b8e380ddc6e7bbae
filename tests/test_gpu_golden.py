"""GPU vs the golden fixtures the REFERENCE produced (tests/golden/make_golden.py):
BASELINE config 0 geometry (B=1, NH=2, S=256, d=64, L=64), both variants,
forward outputs and all gradients. Tolerance as in test_gpu_forward/backward."""
from pathlib import Path

import numpy as np
import pytest

from tests._util import TOL_GRAD, np_, rel, to_dev
from tests.golden.make_golden import load

FIX = sorted(p for p in (Path(__file__).parent / "golden").glob("cfg0_*.npz"))


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIX, ids=[p.stem for p in FIX])
def test_gpu_matches_reference_golden(path):
    import torch

    from paper_2503_14376_b200 import Dims, Variant, chunkwise_backward, chunkwise_forward

    z = load(path)
    B, H, T, L, dqk, dhv, variant = (int(x) for x in z["dims"])
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    inp = to_dev(z["q"], z["k"], z["v"], z["i_pre"], z["f_pre"])
    out = chunkwise_forward(inp, dims, Variant(variant))
    dh = torch.from_numpy(z["dh"]).to("cuda", torch.bfloat16)
    g = chunkwise_backward(inp, dims, Variant(variant), dh, out.states, out.stats, out.saved_states)
    torch.cuda.synchronize()
    errs = {
        "h": rel(np_(out.h_tilde), z["h"]), "C": rel(np_(out.states.C), z["C"]),
        "n": rel(np_(out.states.n), z["n"]), "h_denom": rel(np_(out.stats.h_denom), z["h_denom"]),
    }
    errs.update({n: rel(np_(getattr(g, n)), z[n]) for n in ("dq", "dk", "dv", "d_fpre", "d_ipre")})
    m_err = float(np.abs(np_(out.states.m) - z["m"]).max())
    print(path.stem, {k: f"{e:.2e}" for k, e in errs.items()}, "m", m_err)
    assert m_err < 1e-4
    for n, e in errs.items():
        assert e < (1e-2 if n in ("n", "h_denom") else TOL_GRAD), (n, e)
