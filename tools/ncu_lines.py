"""Per-CUDA-source-line instruction and stall-sample totals from an ncu report
(development tool): python tools/ncu_lines.py REPORT [N]."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg = {}
cur = None
fname = "?"
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] in ("Line No", "Address") and "Instructions Executed" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if "Line No" in d and d.get("Line No", "").isdigit():
        cur = (fname, int(d["Line No"]), d.get("Source", "")[:70])
        ie = d.get("Instructions Executed", "0") or "0"
        ss = d.get("Warp Stall Sampling (All Samples)", "0") or "0"
        try:
            agg[cur] = (float(ie), float(ss))
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k[0][:18]:18s}{k[1]:5d} inst%={100*v[0]/tot:5.1f} stall%={100*v[1]/ts:5.1f}  {k[2]}")
