#!/usr/bin/env python
"""Per-instruction warp-stall breakdown from an ncu source page (--page source --csv --print-source sass).

  python tools/ncu_stalls.py <source.csv> [exec-count-filter]
Prints the stall reasons summed over all instructions (or those executed exactly N times) and the top
instructions with their dominant reasons."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, R = rows[1], rows[2:]
flt = int(sys.argv[2]) if len(sys.argv) > 2 else None
iS, iE = h.index("Source"), h.index("Instructions Executed")
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
per = []
for r in R:
    if not r[iE].isdigit():
        continue
    if flt is not None and int(r[iE]) != flt:
        continue
    d = {h[i][6:]: int(r[i] or 0) for i in cols if (r[i] or "0").isdigit()}
    tot.update(d)
    per.append((sum(d.values()), r[0][-5:], r[iS][:60], d))
T = sum(tot.values())
print("total samples", T)
print({k: f"{v / T:.1%}" for k, v in tot.most_common(10)})
for s, a, src, d in sorted(per, reverse=True)[:25]:
    top = ", ".join(f"{k}:{v}" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{a} {s:5d} {src:60s} {top}")
