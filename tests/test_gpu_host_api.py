"""The C++ host API (include/tfla/mlstm_b200.hpp) end to end: the compiled
tests/host/tfla_host_test binary runs chunkwise_forward/backward,
tfla_forward, the split entry points, the decode step, the frozen forward, the
gated forward (checked bit-exact against the separate output pass inside the
binary) and the fp32-operand forward on the GPU; outputs are compared with the
f64 oracle."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Oracle, bf16_round
from tests._util import TOL_GRAD, TOL_H, make_case, rel

BIN = Path(__file__).resolve().parents[1] / "paper_2503_14376_b200" / "_lib" / "tfla_host_test"


def _bf16_bytes(a):
    return (a.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16).tobytes()


def _from_bf16(buf, shape):
    u = np.frombuffer(buf, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).reshape(shape).astype(np.float64)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_cpp_host_api(tmp_path, variant):
    B, H, T, L, dqk, dhv = 1, 2, 512, 128, 128, 128
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=99 + variant)
    dh = bf16_round(np.random.default_rng(5).standard_normal((B, H, T, dhv)))
    inp = tmp_path / "in.bin"
    inp.write_bytes(_bf16_bytes(q) + _bf16_bytes(k) + _bf16_bytes(v) + ip.astype(np.float32).tobytes()
                    + fp.astype(np.float32).tobytes() + _bf16_bytes(dh))
    outp = tmp_path / "out.bin"
    r = subprocess.run([str(BIN), f"{B},{H},{T},{L},{dqk},{dhv},{variant}", str(inp), str(outp)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    raw = outp.read_bytes()
    sizes = [("h", (B, H, T, dhv), 2), ("C_final", (B, H, dqk, dhv), 4), ("dq", (B, H, T, dqk), 2),
             ("dk", (B, H, T, dqk), 2), ("dv", (B, H, T, dhv), 2), ("d_fpre", (B, H, T), 4),
             ("d_ipre", (B, H, T), 4), ("h_tiled", (B, H, T, dhv), 2), ("h_split", (B, H, T, dhv), 2),
             ("dq_split", (B, H, T, dqk), 2), ("dk_split", (B, H, T, dqk), 2), ("dv_split", (B, H, T, dhv), 2),
             ("h_decode", (B, H, T, dhv), 2), ("C_decode", (B, H, dqk, dhv), 4), ("h_frozen", (B, H, T, dhv), 2),
             ("h_f32", (B, H, T, dhv), 4)]
    got, off = {}, 0
    for name, shape, es in sizes:
        n = int(np.prod(shape)) * es
        chunk = raw[off:off + n]
        off += n
        got[name] = _from_bf16(chunk, shape) if es == 2 else np.frombuffer(chunk, np.float32).reshape(shape).astype(np.float64)
    orc = Oracle()
    f = orc.forward(q, k, v, ip, fp, L, variant)
    g = orc.backward(q, k, v, ip, fp, dh, f["C"], f["m"], f["m_comb"], f["h_denom"], L, variant)
    assert rel(got["h"], f["h"]) < TOL_H
    assert rel(got["h_tiled"], f["h"]) < TOL_H
    assert rel(got["C_final"], f["C"][:, :, -1]) < TOL_H
    assert rel(got["h_split"], f["h"]) < TOL_H
    for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
        assert rel(got[n], g[n]) < TOL_GRAD, n
    for n in ("dq", "dk", "dv"):
        assert rel(got[n + "_split"], g[n]) < TOL_GRAD, n
    # decode (recurrent_step, fp32 state) over the same sequence
    assert rel(got["h_decode"], f["h"]) < TOL_H
    assert rel(got["C_decode"], f["C"][:, :, -1]) < TOL_H
    # chunkwise_forward_frozen (C++ mirror) under the forward's own stats
    assert rel(got["h_frozen"], f["h"]) < TOL_H
    # chunkwise_forward_f32 (C++ mirror): fp32 operands, reference precision
    assert rel(got["h_f32"], f["h"]) < 1e-4
