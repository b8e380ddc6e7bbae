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
a = np.loadtxt("/tmp/trb.txt", max_rows=512).astype(np.int64)
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
# epilogue events (thread et 0 of CTA 0), rows 512.. : [0] tile start, [1] scores ready,
# [2] gating done, [3+3q] group q TMEM ready, [4+3q] rows landed, [5+3q] group stored
lines = open("/tmp/trb.txt").read().splitlines()
if len(lines) > 512:
    e = np.array([[int(x) for x in ln.split()] for ln in lines[512:576]], dtype=np.int64)
    ng = 8
    sel = e[1:11]
    print("epilogue per tile (tiles 1..10, cycles): interval", np.diff(e[1:12, 0]).mean().round())
    print("  wait scores", (sel[:, 1] - sel[:, 0]).mean().round(), "gating", (sel[:, 2] - sel[:, 1]).mean().round())
    prev = sel[:, 2]
    for q in range(ng):
        tm, rw, dn = sel[:, 3 + 3 * q], sel[:, 4 + 3 * q], sel[:, 5 + 3 * q]
        print(f"  group {q}: wait TMEM {(tm - prev).mean():7.0f}  wait rows {(rw - tm).mean():6.0f}  drain+store {(dn - rw).mean():6.0f}")
        prev = dn
