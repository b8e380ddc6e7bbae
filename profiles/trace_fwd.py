import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2503_14376_b200 import Dims, Variant, SequenceInputs, chunkwise_forward
B,H,T = int(os.environ.get("TB",8)), 8, int(os.environ.get("TT",8192))
dqk, dhv = 256, 512
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
inp = SequenceInputs(mk(B,H,T,dqk), mk(B,H,T,dqk), mk(B,H,T,dhv), torch.randn(B,H,T,device="cuda",generator=g), torch.randn(B,H,T,device="cuda",generator=g))
d = Dims(T,128,dqk,dhv,H,B)
for _ in range(3): chunkwise_forward(inp, d, Variant.Exp, all_states=False)
torch.cuda.synchronize()
names = ["mma.pre_sbv","mma.sbv_go","mma.cready","mma.qc_issued","mma.cupd_issued","mma.s_go","mma.S_issued",
         "C.pre_cfull","C.cfull","C.rt_done","T.q0_loop","T.q0_fence","T.q1_loop","T.q1_fence","HS.pre_hfull","HS.hfull",
         "T.q_wait0","T.q_got","T.v_wait","T.v_got","T.v_done","T.q1_got","HS.drained","HS.gated",
         "P.qc0_pre","P.qc0_go","P.cu0_pre","P.cu0_go","P.s0_pre","P.s0_go","P.slast_pre","P.slast_go"]
for cta in (0, int(os.environ.get("CTA2", 200))):
    os.environ["TFLA_TRACE_FWD"] = f"/tmp/tr{cta}.txt"; os.environ["TFLA_TRACE_CTA"] = str(cta)
    chunkwise_forward(inp, d, Variant.Exp, all_states=False); torch.cuda.synchronize()
    del os.environ["TFLA_TRACE_FWD"]
    a = np.loadtxt(f"/tmp/tr{cta}.txt").astype(np.int64)
    NC = a.shape[0]
    base = a[0,0]
    print(f"== CTA {cta}: total {a[NC-2,6]-a[0,0]} cyc for {NC-2} chunks -> {(a[NC-2,6]-a[1,6])/(NC-3):.0f} cyc/chunk (S_issued to S_issued)")
    ks = range(4, NC-4)
    # print, relative to mma.pre_cready of chunk k, the mean time of each event
    for e, n in enumerate(names):
        if n == '-': continue
        rel = np.array([a[k, e] - a[k, 0] for k in ks])
        print(f"  {n:16s} mean {rel.mean():8.0f}  min {rel.min():8.0f} max {rel.max():8.0f}")
