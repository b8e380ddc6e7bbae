"""Per-CUDA-source-line warp-stall shares of an ncu report (needs -lineinfo and
--import-source): python profiles/ncu_lines.py rep.ncu-rep [top] [launch]."""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    args += ["--launch-skip", sys.argv[3], "--launch-count", "1"]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
acc = defaultdict(float)
text = {}
fname, hdr, line = "?", None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        line = (fname, r[0])
        text[line] = r[1]
    try:
        acc[line] += float(r[4] or 0)
    except ValueError:
        pass
tot = sum(acc.values()) or 1
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot:6.3f} {k[0]}:{k[1]:>4} {text.get(k, '')[:100].strip()}")
