"""Cost of the cell output epilogue at the 7B shape (B=8, NH=8, S=8192, dqk=256,
dhv=512, L=128): plain forward, forward + separate output pass, and the gated
forward with the epilogue fused into K12's H drain (cluster DSMEM row sums).
CUDA events around 20 replays each; prints ms per call."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2503_14376_b200 import (Dims, SequenceInputs, Variant, chunkwise_forward,  # noqa: E402
                                   chunkwise_forward_gated, output_norm_gate)

B, H, T, L, dqk, dhv = (int(x) for x in os.environ.get("OUT_SHAPE", "8,8,8192,128,256,512").split(","))
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)  # noqa: E731
inp = SequenceInputs(mk(B, H, T, dqk), mk(B, H, T, dqk), mk(B, H, T, dhv), torch.randn(B, H, T, device="cuda", generator=g),
                     torch.randn(B, H, T, device="cuda", generator=g))
o = mk(B, H, T, dhv)
gamma = torch.randn(H, dhv, device="cuda", generator=g)
d = Dims(T, L, dqk, dhv, H, B)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


plain = lambda: chunkwise_forward(inp, d, Variant.Exp, all_states=False)  # noqa: E731
sep = lambda: output_norm_gate(plain().h_tilde, o, gamma, 1e-6)  # noqa: E731
fused = lambda: chunkwise_forward_gated(inp, d, Variant.Exp, o, gamma, 1e-6, all_states=False)  # noqa: E731
print(f"forward                    {t(plain):.3f} ms")
print(f"forward + output pass      {t(sep):.3f} ms")
print(f"gated forward (default: separate pass)  {t(fused):.3f} ms")
os.environ["TFLA_FUSED_OUT"] = "1"
print(f"gated forward (TFLA_FUSED_OUT=1, fused into K12's H drain)  {t(fused):.3f} ms")
