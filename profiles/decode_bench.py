"""Decode (recurrent step) throughput on one B200: tfla_recurrent_step at the
7B head shape (dqk=256, dhv=512), B*NH = 64 heads, T = 1 and T = 16 steps per
launch. The step is HBM-bound on the fp32 state: per launch C is read and
written once (2 * 64 * 256 * 512 * 4 B = 67 MB) plus n, m and the T-step
q/k/v/h vectors. Prints one JSON line; CUDA-event timing after warm-up."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_14376_b200 import Dims, MemoryState, SequenceInputs, Variant, recurrent_step  # noqa: E402

peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
B, NH, dqk, dhv = 8, 8, 256, 512
res = {}
for T in [int(x) for x in __import__("os").environ.get("DEC_T", "1,16").split(",")]:
    g = torch.Generator(device="cuda").manual_seed(T)
    mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
    inp = SequenceInputs(mk(B, NH, T, dqk), mk(B, NH, T, dqk), mk(B, NH, T, dhv),
                         torch.randn(B, NH, T, device="cuda", generator=g),
                         torch.randn(B, NH, T, device="cuda", generator=g))
    d = Dims(T, 1, dqk, dhv, NH, B)
    st = MemoryState.zero(d)
    for _ in range(5):
        recurrent_step(inp, d, Variant.Exp, st)
    torch.cuda.synchronize()
    # device time per launch: 20 launches captured in one CUDA graph (no host
    # launch overhead between them), replayed; eager per-call time beside it
    n_g = 20
    gr = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=cap):
        for _ in range(n_g):
            recurrent_step(inp, d, Variant.Exp, st)
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (reps * n_g) * 1e3
    n = 50
    e0.record()
    for _ in range(n):
        recurrent_step(inp, d, Variant.Exp, st)
    e1.record()
    torch.cuda.synchronize()
    us_eager = e0.elapsed_time(e1) / n * 1e3
    nbytes = B * NH * (2 * dqk * dhv * 4 + 2 * dqk * 4 + 8 + T * (2 * dqk * 2 + 2 * dhv * 2 + 8))
    res[f"T{T}"] = {"us_per_launch": round(us, 2), "us_per_call_eager": round(us_eager, 2),
                    "tokens_per_s": B * T / (us * 1e-6),
                    "gbs": round(nbytes / (us * 1e-6) / 1e9, 1),
                    "hbm_frac": round(nbytes / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3)}
print(json.dumps({"decode": "mLSTMexp recurrent_step B=8 NH=8 dqk=256 dhv=512", **res}))

# output epilogue at the 7B h shape: read h_tilde + o_pre, write h (3 x 537 MB)
from paper_2503_14376_b200 import output_norm_gate  # noqa: E402

T = 8192
ht = torch.randn(B, NH, T, dhv, device="cuda").to(torch.bfloat16)
op = torch.randn(B, NH, T, dhv, device="cuda").to(torch.bfloat16)
gm = torch.randn(NH, dhv, device="cuda")
for _ in range(3):
    output_norm_gate(ht, op, gm)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    output_norm_gate(ht, op, gm)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nb = 3 * ht.numel() * 2
print(json.dumps({"output_norm_gate": "B=8 NH=8 S=8192 dhv=512", "ms": round(ms, 4),
                  "gbs": round(nb / (ms * 1e-3) / 1e9, 1), "hbm_frac": round(nb / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 3)}))
