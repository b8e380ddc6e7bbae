import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from tests._util import make_case, to_dev
from paper_2503_14376_b200 import Dims, Variant, chunkwise_forward, chunkwise_backward, run_recurrent, output_norm_gate
for (B,H,T,L,dqk,dhv), env in [((1,2,256,64,64,64), {}), ((1,1,512,128,256,256), {"TFLA_FORCE_FUSED_FWD": "1"}), ((1,1,384,128,128,128), {"TFLA_NO_FUSED_FWD": "1", "TFLA_NO_FUSED_BWD": "1"})]:
    for k_, v_ in env.items(): os.environ[k_] = v_
    q,k,v,ip,fp = make_case(B,H,T,dqk,dhv,seed=1)
    inp = to_dev(q,k,v,ip,fp)
    d = Dims(T=T,L=L,d_qk=dqk,d_hv=dhv,n_head=H,n_batch=B)
    for var in (0,1):
        o = chunkwise_forward(inp, d, Variant(var))
        g = chunkwise_backward(inp, d, Variant(var), torch.randn(B,H,T,dhv,device="cuda").to(torch.bfloat16), o.states, o.stats, o.saved_states)
    for k_ in env: del os.environ[k_]
    torch.cuda.synchronize()
    print("ok", (B,H,T,L,dqk,dhv), flush=True)
tr = run_recurrent(inp, Dims(T=T, L=1, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B), Variant.Exp)
h = output_norm_gate(o.h_tilde, o.h_tilde, torch.ones(H, dhv, device="cuda"))
torch.cuda.synchronize(); print("all ok")
