"""Summarise an ncu report: per kernel duration, DRAM/L2 throughput, tensor
pipe, stall reasons, and the top stalled SASS instructions."""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
def col(r, k):
    return r[hdr.index(k)] if k in hdr else "?"
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]
for i, r in enumerate(data):
    print(f"== [{i}] {col(r, 'Kernel Name')[:80]}")
    for k in keys:
        if k in hdr:
            print(f"   {k:90s} {col(r, k)} {units[hdr.index(k)]}")
    st = []
    for j, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st.append((float(r[j].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{n} {v / tot:.0%}" for v, n in st[:6]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(i), "--launch-count", "1"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) < 3:
        continue
    sh = srows[1]
    sd = [x for x in srows[2:] if len(x) == len(sh) and x[0] != "Address"]
    iss = sh.index("Warp Stall Sampling (All Samples)")
    isrc = sh.index("Source")
    f = lambda x: float(x) if x.replace(".", "").isdigit() else 0.0
    tot = sum(f(x[iss]) for x in sd) or 1
    seen = set()
    for x in sorted(sd, key=lambda x: -f(x[iss])):
        if x[0] in seen:
            continue
        seen.add(x[0])
        print(f"   {f(x[iss]) / tot:6.3f} {x[isrc][:100]}")
        if len(seen) >= ntop:
            break
