"""Per-instruction stall attribution from an ncu source-page CSV
(ncu -i R --page source --csv --print-source sass): top instructions for one
stall reason, and the reason totals by opcode."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15


def f(r, k):
    try:
        return float(r[col[k]] or 0)
    except ValueError:
        return 0.0


reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {k: sum(f(r, k) for r in data) for k in reasons}
all_s = sum(tot.values())
print("reason totals:", ", ".join(f"{k[6:]} {v / all_s:.1%}" for k, v in
                                   sorted(tot.items(), key=lambda kv: -kv[1]) if v > 0))
byop = collections.Counter()
for r in data:
    op = r[col["Source"]].split()
    op = [t for t in op if not t.startswith("@")]
    byop[op[0].split(".")[0] if op else "?"] += f(r, reason)
print(f"{reason} by opcode:", ", ".join(f"{k} {v / max(tot[reason], 1):.0%}" for k, v in
                                        byop.most_common(8)))
for r in sorted(data, key=lambda r: -f(r, reason))[:n]:
    print(r[col["Address"]][-5:], f"{f(r, reason) / all_s:6.2%}", r[col["Source"]].strip()[:80])
