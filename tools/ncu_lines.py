"""Per-source-line share of executed instructions and stall samples of one
kernel in an .ncu-rep, joining ncu's per-address counts with the line table
of `nvdisasm --print-line-info`.
usage: python tools/ncu_lines.py report.ncu-rep cubin mangled_kernel_name [n]"""
import collections, csv, io, re, subprocess, sys

rep, cubin, fn = sys.argv[1], sys.argv[2], sys.argv[3]
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 30
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True,
                     text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(f".text.{fn}:"))
cur, off2line = "?", {}
for l in dis[start + 1:]:
    if l.startswith(".text.") or "\t.section" in l:
        break
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; ix = {n: i for i, n in enumerate(h)}
data = rows[2:]
base = int(data[0][ix["Address"]], 16)
inst, stall = collections.Counter(), collections.Counter()
ti = ts = 0
for r in data:
    line = off2line.get(int(r[ix["Address"]], 16) - base, "?")
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    inst[line] += n; stall[line] += s; ti += n; ts += s
print(f"mapped {len(off2line)} instructions")
for k, v in inst.most_common(ntop):
    print(f"{100 * v / ti:5.1f}% inst  {100 * stall[k] / max(ts, 1):5.1f}% stall  {k}")
