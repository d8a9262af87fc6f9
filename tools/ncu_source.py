#!/usr/bin/env python
"""Per-instruction breakdown of an ncu --set full --import-source capture: shared-memory wavefronts per
unit of work, stall reasons of the hottest loop, and the instruction mix.

  python tools/ncu_source.py <report.ncu-rep> <units-of-work>
"""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = rows[2:]
iv = lambda r, k: int(float(r[ix[k]] or 0))
wf = sum(iv(r, "L1 Wavefronts Shared") for r in data)
wfi = sum(iv(r, "L1 Wavefronts Shared Ideal") for r in data)
print(f"shared wavefronts per unit: {wf / units:.1f} (ideal {wfi / units:.1f})")
samples = sum(iv(r, "Warp Stall Sampling (All Samples)") for r in data)
by_exec = collections.Counter()
for r in data:
    by_exec[iv(r, "Instructions Executed")] += iv(r, "Warp Stall Sampling (All Samples)")
hot_exec = by_exec.most_common(1)[0][0]
hot = [r for r in data if iv(r, "Instructions Executed") == hot_exec]
print(f"samples {samples}; hottest block executes {hot_exec}x, {len(hot)} instrs, "
      f"{by_exec[hot_exec] / samples:.0%} of samples")
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = collections.Counter()
for r in hot:
    for k in reasons:
        tot[k] += iv(r, k)
s = sum(tot.values())
print("hot-block stalls:", ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in tot.most_common(9)))
op = lambda src: (src.split()[1] if src.startswith("@") else src.split()[0])
mix = collections.Counter(op(r[ix["Source"]]) for r in hot)
print("hot-block mix:", dict(mix.most_common(14)))
hw = collections.Counter()
for r in hot:
    hw[op(r[ix["Source"]])] += iv(r, "L1 Wavefronts Shared")
print("hot-block wavefronts by opcode (per execution):", {k: v / hot_exec for k, v in hw.most_common(6) if v})
