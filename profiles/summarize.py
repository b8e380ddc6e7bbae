"""Turn a round's gpurun_out/ profile bundle into the committed summaries:
profiles/<tag>_launches.csv, <tag>_ncu_summary.md, <tag>_bench.json, traffic.json."""
import csv
import json
import shutil
import sys
from pathlib import Path

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = Path(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out")
dst = Path(__file__).resolve().parent
shutil.copy(src / "launches.csv", dst / f"{tag}_launches.csv")
bench = json.loads((src / "bench.json").read_text().strip().splitlines()[-1])
(dst / f"{tag}_bench.json").write_text(json.dumps(bench, indent=1) + "\n")

rows = list(csv.reader(open(src / "launches.csv")))
hdr, per = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("::")[-1].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "usecond": 1e-3,
                 "nsecond": 1e-6, "msecond": 1}.get(unit, 1)
        per.setdefault((int(d["ID"]), name), {})[d["Metric Name"]] = v * scale
names = {"state_scan_kernel<0, 64>": "state_scan_fwd", "state_scan_kernel<1, 64>": "state_scan_bwd",
         "fwd_parallel_kernel<128>": "fwd_parallel", "fwd_parallel_kernel<256>": "fwd_parallel",
         "bwd_fused_kernel": "bwd_fused", "fwd_fused_kernel<2>": "fwd_fused",
         "bwd_parallel_kernel<0, 256>": "bwd_dq", "bwd_parallel_kernel<1, 256>": "bwd_dk",
         "bwd_parallel_kernel<2, 256>": "bwd_dv", "state_scan2_kernel<0>": "state_scan_fwd"}
traffic = {}
lines = ["| # | kernel | ncu duration ms | DRAM read GB | DRAM write GB | DRAM GB/s |", "|---|---|---|---|---|---|"]
for (i, k), m in sorted(per.items()):
    t = m.get("gpu__time_duration.sum", 0)
    rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
    lines.append(f"| {i} | {k} | {t:.3f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | {(rd + wr) / (t / 1e3) / 1e9 if t else 0:.0f} |")
    if k in names:
        traffic[names[k]] = rd + wr
old = json.loads((dst / "traffic.json").read_text()) if (dst / "traffic.json").exists() else {}
old.setdefault("exp", {})[sys.argv[3] if len(sys.argv) > 3 else "128"] = traffic
json.dump(old, open(dst / "traffic.json", "w"), indent=1)
full = (src / "prof_full.txt").read_text() if (src / "prof_full.txt").exists() else ""
md = [f"# {tag} -- ncu summary (7B shape B=8 NH=8 S=8192 dqk=256 dhv=512, L=128, mLSTMexp, one fwd+bwd step)", "",
      "Produced by `profiles/run_round_profile.sh` under gpurun (1 B200) and `profiles/summarize.py`.",
      "Launch list: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
      "--clock-control none` (cold-cache, serialised: compare kernel shares with bench.py's live CUDA-event "
      "times, not absolutes).", "", "## Launch list (one step)", ""] + lines + [
      "", "## Bench line of the same build (live CUDA events, not under ncu)", "",
      f"ms/step {bench['ms_per_step']:.3f}, {bench['value'] / 1e6:.2f} M tokens/s, "
      f"{bench['tensor_peak_frac']:.3f} of sustained bf16 peak; per-kernel ms: "
      + ", ".join(f"{k} {v['ms']}" for k, v in bench["kernels"].items()), "",
      "## `--set full` captures (tcgen05 kernels): throughput, pc-sampling stalls, top stalled SASS", "", "```", full.strip(), "```", ""]
(dst / f"{tag}_ncu_summary.md").write_text("\n".join(md))
print("\n".join(lines))
