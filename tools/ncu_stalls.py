"""Summarise an .ncu-rep: headline metrics, stall split, hottest SASS lines.
usage: python tools/ncu_stalls.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for w in want:
    if w in h:
        print(f"{w:60s} {v[h.index(w)]}")
st = {n: float(v[i] or 0) for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not n.endswith("not_issued")}
tot = sum(st.values()) or 1
for n, x in sorted(st.items(), key=lambda t: -t[1])[:8]:
    print(f"  {n.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {100 * x / tot:5.1f} %")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
data = rows[2:]
key = "Warp Stall Sampling (All Samples)"
top = sorted(range(len(data)), key=lambda j: -int(data[j][ix[key]] or 0))[:ntop]
kinds = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for j in top:
    r = data[j]
    worst = max(kinds, key=lambda k: int(r[ix[k]] or 0))
    print(f"{r[ix[key]]:>7s} {worst:18s} {r[ix['Source']].strip()[:70]}")
