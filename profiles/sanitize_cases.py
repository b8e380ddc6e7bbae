import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from tests._util import make_case, to_dev
from paper_2503_14376_b200 import (Dims, Variant, chunkwise_forward, chunkwise_backward, chunkwise_forward_gated,
                                   run_recurrent, output_norm_gate)
CASES = [((1, 2, 256, 64, 64, 64), {}),
         ((1, 1, 512, 128, 256, 256), {"TFLA_FORCE_FUSED_FWD": "1"}),
         ((1, 1, 384, 128, 128, 128), {"TFLA_NO_FUSED_FWD": "1", "TFLA_NO_FUSED_BWD": "1"}),
         ((1, 1, 512, 256, 256, 512), {}),                                   # wide split kernels, L = 256
         ((1, 1, 384, 128, 128, 64), {"TFLA_SCAN32": "1", "TFLA_NO_FUSED_FWD": "1"})]  # 32-column scans
for (B, H, T, L, dqk, dhv), env in CASES:
    for k_, v_ in env.items(): os.environ[k_] = v_
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=1)
    inp = to_dev(q, k, v, ip, fp)
    d = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    for var in (0, 1):
        o = chunkwise_forward(inp, d, Variant(var))
        g = chunkwise_backward(inp, d, Variant(var), torch.randn(B, H, T, dhv, device="cuda").to(torch.bfloat16),
                               o.states, o.stats, o.saved_states)
    for k_ in env: del os.environ[k_]
    torch.cuda.synchronize()
    print("ok", (B, H, T, L, dqk, dhv), env, flush=True)
# gated forward with the epilogue fused into K12 (clusters of 2 x-tile CTAs, DSMEM row sums)
os.environ["TFLA_FORCE_FUSED_FWD"] = "1"
os.environ["TFLA_FUSED_OUT"] = "1"
B, H, T, dqk, dhv = 1, 2, 512, 256, 256
inp = to_dev(*make_case(B, H, T, dqk, dhv, seed=2))
o_pre = torch.randn(B, H, T, dhv, device="cuda").to(torch.bfloat16)
for var in (0, 1):
    chunkwise_forward_gated(inp, Dims(T, 128, dqk, dhv, H, B), Variant(var), o_pre, torch.ones(H, dhv, device="cuda"))
del os.environ["TFLA_FUSED_OUT"], os.environ["TFLA_FORCE_FUSED_FWD"]
torch.cuda.synchronize()
print("ok gated", flush=True)
# decode: 4 column slices per head (one cluster), 20 steps (two staging blocks)
B, H, T, dqk, dhv = 1, 2, 20, 128, 256
inp = to_dev(*make_case(B, H, T, dqk, dhv, seed=3))
for var in (0, 1):
    tr = run_recurrent(inp, Dims(T=T, L=1, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), Variant(var))
h = output_norm_gate(o.h_tilde, o.h_tilde, torch.ones(o.h_tilde.shape[1], o.h_tilde.shape[3], device="cuda"))
torch.cuda.synchronize(); print("all ok")
