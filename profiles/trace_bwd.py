import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2503_14376_b200 import Dims, Variant, SequenceInputs, chunkwise_forward, chunkwise_backward
B,H,T = 8, 8, 8192
dqk, dhv = 256, 512
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
inp = SequenceInputs(mk(B,H,T,dqk), mk(B,H,T,dqk), mk(B,H,T,dhv), torch.randn(B,H,T,device="cuda",generator=g), torch.randn(B,H,T,device="cuda",generator=g))
d = Dims(T,128,dqk,dhv,H,B)
dh = mk(B,H,T,dhv)
o = chunkwise_forward(inp, d, Variant.Exp, all_states=False)
for _ in range(3): chunkwise_backward(inp, d, Variant.Exp, dh, o.states, o.stats, o.saved_states)
torch.cuda.synchronize()
os.environ["TFLA_TRACE_BWD"] = "/tmp/trb.txt"
chunkwise_backward(inp, d, Variant.Exp, dh, o.states, o.stats, o.saved_states); torch.cuda.synchronize()
a = np.loadtxt("/tmp/trb.txt").astype(np.int64)
per_tile = 68
t0 = a[0,1]
print("stage: acq_wait(empty) | tma+issue latency (take_done - acq_done) | mma waiting (take_done - take_pre)")
for gi in list(range(per_tile, per_tile + 80)):
    acq_pre, acq, tpre, tdone = a[gi]
    print(f"{gi:4d} t={acq - t0:8d}  empty_wait {acq-acq_pre:6d}  lat {tdone-acq:6d}  mma_wait {tdone-tpre:6d}")
tiles = [a[k*per_tile,1] for k in range(1, 6)]
print("cycles per tile:", np.diff(tiles))
# aggregate over tiles 1..6
rows = np.arange(per_tile, 7 * per_tile)
acq_pre, acq, tpre, tdone = a[rows].T
print("mean empty_wait", (acq - acq_pre).mean(), "mean latency", (tdone - acq).mean(), "mean mma_wait", (tdone - tpre).mean())
ls = rows % per_tile
for name, sel in (("S", ls < 4), ("dS", (ls >= 4) & (ls < 12)), ("groups", ls >= 12)):
    print(name, "lat", (tdone - acq)[sel].mean(), "mma_wait", (tdone - tpre)[sel].mean(), "empty_wait", (acq - acq_pre)[sel].mean())
