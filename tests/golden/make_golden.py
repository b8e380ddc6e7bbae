"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libmlstm_ref.so,
the unmodified reference sources compiled by oracle/Makefile). Run in the build
container (where /root/reference exists):  python tests/golden/make_golden.py

Inputs come from the reference RNG (make_inputs(dims, Rng(seed), 1.0, 1.0),
core.cpp:127-143; dH from the same stream), then q/k/v/dH are rounded to bf16
and i/f to fp32 so that the B200 kernels consume exactly the values the
reference computed on. Outputs are the reference's f64 chunkwise_forward /
chunkwise_backward (and tfla_* with the given block config) results.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Reference, bf16_round  # noqa: E402

CASES = {
    # name: (B, H, T, L, dqk, dhv, seed, blocks)
    "cfg0": (1, 2, 256, 64, 64, 64, 1, None),          # BASELINE config 0 (oracle case)
    "small": (2, 2, 32, 8, 8, 12, 3, None),             # CPU-oracle-only geometry
}


def load(path):
    """Load a fixture: bf16 patterns -> f64 values."""
    z = np.load(path)
    out = {k: z[k] for k in z.files}
    for k in ("q", "k", "v", "dh"):
        out[k] = (out[k].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    for k in ("i_pre", "f_pre"):
        out[k] = out[k].astype(np.float64)
    return out


def main():
    ref = Reference()
    out_dir = Path(__file__).resolve().parent
    for name, (B, H, T, L, dqk, dhv, seed, blocks) in CASES.items():
        q, k, v, ip, fp = ref.make_inputs(B, H, T, dqk, dhv, seed=seed, scale=1.0, gate_scale=1.0)
        dh = ref.normals(seed + 100, 0, B * H * T * dhv).reshape(B, H, T, dhv)
        q, k, v, dh = (bf16_round(x) for x in (q, k, v, dh))
        ip = ip.astype(np.float32).astype(np.float64)
        fp = fp.astype(np.float32).astype(np.float64)
        for variant in (0, 1):
            f = ref.forward(q, k, v, ip, fp, L, variant, blocks=blocks)
            g = ref.backward(q, k, v, ip, fp, dh, f["C"], f["n"], f["m"], f["m_comb"], f["h_denom"],
                             L, variant, blocks=blocks)
            tag = f"{name}_{'exp' if variant == 0 else 'sig'}"
            # bf16 inputs stored as their raw 16-bit patterns, outputs as fp32
            b16 = lambda x: (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
            f32 = lambda x: x.astype(np.float32)
            np.savez_compressed(
                out_dir / f"{tag}.npz",
                dims=np.array([B, H, T, L, dqk, dhv, variant]),
                q=b16(q), k=b16(k), v=b16(v), dh=b16(dh), i_pre=f32(ip), f_pre=f32(fp),
                h=f32(f["h"]), C=f32(f["C"]), n=f32(f["n"]), m=f32(f["m"]),
                m_comb=f32(f["m_comb"]), h_denom=f32(f["h_denom"]),
                dq=f32(g["dq"]), dk=f32(g["dk"]), dv=f32(g["dv"]),
                d_fpre=f32(g["d_fpre"]), d_ipre=f32(g["d_ipre"]),
            )
            print("wrote", tag)


if __name__ == "__main__":
    main()
