"""Summarise an ncu report: key metrics + hot SASS regions (development tool)."""
import csv, re, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    print("kernel:", d.get("Kernel Name", ("?",))[0][:90])
    keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__cycles_elapsed.avg"]
    for k in keys:
        if k in d: print(f"  {k} = {d[k][0]} {d[k][1]}")
    st = [(k, float(v[0])) for k, v in d.items() if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", k)]
    st.sort(key=lambda x: -x[1])
    print("  stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in st[:8]))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = rows[1]; ia = h.index("Instructions Executed"); isamp = h.index("Warp Stall Sampling (All Samples)")
    data = [(r[1], int(r[ia] or 0), int(r[isamp] or 0)) for r in rows[2:] if len(r) > ia]
    tot = sum(x[1] for x in data); ts = sum(x[2] for x in data) or 1
    out = []; cur = None; start = 0; acc = sacc = 0
    for i, (s, e, sm) in enumerate(data + [("", -1, 0)]):
        if e != cur:
            if cur is not None: out.append((start, i - 1, cur, acc, sacc, data[start][0].strip()[:60]))
            cur, start, acc, sacc = e, i, 0, 0
        acc += max(e, 0); sacc += sm
    out.sort(key=lambda x: -x[3])
    for o in out[:int(sys.argv[2])]:
        print(f"  [{o[0]:4d}-{o[1]:4d}] n={o[1]-o[0]+1:3d} exec={o[2]:>10d} inst%={o[3]/tot*100:5.1f} stall%={o[4]/ts*100:5.1f} {o[5]}")
