"""Summarise a TFLA_TRACE_SCAN dump of state_scan.cu (CTA (0,0,0)):
per-stage producer issue / transform in / transform out / MMA start, and
per-chunk emit start / emit end / accumulator ready / fold done (clock64)."""
import sys

import numpy as np

lines = open(sys.argv[1]).read().splitlines()
st = np.array([[int(x) for x in ln.split()] for ln in lines[:256]], dtype=np.int64)
ch = np.array([[int(x) for x in ln.split()] for ln in lines[256:384]], dtype=np.int64)
nst = int((st[:, 0] > 0).sum())
nch = int((ch[:, 0] > 0).sum())
st, ch = st[:nst], ch[:nch]
t0 = st[0, 0]
print(f"stages {nst}, chunks {nch}, total {st[-1, 3] - t0} cyc, per stage {(st[-1, 3] - st[0, 3]) / max(nst - 1, 1):.0f}")
d = lambda a, b: (b - a)
print("stage: TMA latency (issue->transform sees full) mean", np.mean(d(st[:, 0], st[:, 1])).round(),
      "| transform time", np.mean(d(st[:, 1], st[:, 2])).round(), "| transform->MMA", np.mean(d(st[:, 2], st[:, 3])).round())
print("stage issue interval", np.mean(np.diff(st[:, 0])).round(), " MMA interval", np.mean(np.diff(st[:, 3])).round())
print("chunk: emit", np.mean(d(ch[:, 0], ch[:, 1])).round(), "| wait acc", np.mean(d(ch[:, 1], ch[:, 2])).round(),
      "| fold", np.mean(d(ch[:, 2], ch[:, 3])).round(), "| chunk interval", np.mean(np.diff(ch[:, 0])).round())
for i in range(min(6, nst)):
    print("  st", i, (st[i] - t0).tolist())
for i in range(min(4, nch)):
    print("  ch", i, (ch[i] - t0).tolist())
if (ch[:, 4] > 0).any():
    print("emit split: wait C tile", np.mean(ch[:, 4] - ch[:, 0]).round(), "| dot", np.mean(ch[:, 5] - ch[:, 4]).round(),
          "| store-wait+bar1", np.mean(ch[:, 6] - ch[:, 5]).round(), "| staging+bar2", np.mean(ch[:, 7] - ch[:, 6]).round(),
          "| TMA store issue", np.mean(ch[:, 1] - ch[:, 7]).round())
