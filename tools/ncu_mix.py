"""Instruction mix (executed warp instructions by opcode) of an .ncu-rep.
usage: python tools/ncu_mix.py report.ncu-rep [units_for_per_unit]"""
import collections, csv, io, subprocess, sys
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; ix = {n: i for i, n in enumerate(h)}
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cnt = collections.Counter(); tot = 0
for r in rows[2:]:
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    cnt[op] += n; tot += n
print("total", tot, "per unit", tot / units)
for op, n in cnt.most_common(24):
    print(f"{op:10s} {100 * n / tot:5.1f}%  {n / units:8.1f}")
