"""Per-source-line warp-stall samples of one kernel in an ncu report
(ncu --page source --print-source cuda,sass). usage: ncu_lines_src.py rep launch_idx [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
data = rows[rows.index(hdr) + 1:]
i_line, i_src, i_st = 0, 1, hdr.index("Warp Stall Sampling (All Samples)")
acc = defaultdict(float)
text = {}
cur = None
for r in data:
    if len(r) < len(hdr):
        continue
    if r[0].strip():
        cur = int(r[0]) if r[0].isdigit() else cur
        text[cur] = r[1]
    try:
        acc[cur] += float(r[i_st] or 0)
    except ValueError:
        pass
tot = sum(acc.values()) or 1
for ln, v in sorted(acc.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot:6.3f}  L{ln}: {text.get(ln, '')[:110]}")
