#!/usr/bin/env python
"""Static issue model of a kernel's hot block: decode the control bits (stall count, yield, barriers) of
every SASS instruction from `cuobjdump -sass` and report, per basic block that holds MMAs, the instruction
count and the sum of stall cycles (the single-warp issue time of that block).

  python tools/sass_stalls.py paper_2505_22179_b200/libw4a16.so <mangled-kernel-name> [--dump]
"""
import re
import subprocess
import sys


def decode(so, fun):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, so], capture_output=True, text=True).stdout.split("\n")
    ins = []
    i = 0
    while i < len(out):
        m = re.match(r"\s+/\*([0-9a-f]{4,6})\*/\s+(.*?);\s+/\* (0x[0-9a-f]{16}) \*/", out[i])
        if m:
            lo = int(m.group(3), 16)
            hi = int(re.search(r"/\* (0x[0-9a-f]{16}) \*/", out[i + 1]).group(1), 16)
            w = (hi << 64) | lo
            ins.append((int(m.group(1), 16), m.group(2).strip(), (w >> 105) & 0xF, (w >> 109) & 1))
            i += 2
            continue
        i += 1
    return ins


def blocks(ins):
    # split at branch targets and after branches
    targets = set()
    for a, t, _, _ in ins:
        m = re.search(r"BRA\s.*?(0x[0-9a-f]+)", t)
        if m:
            targets.add(int(m.group(1), 16))
    cur = []
    for x in ins:
        if x[0] in targets and cur:
            yield cur
            cur = []
        cur.append(x)
        if "BRA" in x[1] or "EXIT" in x[1]:
            yield cur
            cur = []
    if cur:
        yield cur


if __name__ == "__main__":
    ins = decode(sys.argv[1], sys.argv[2])
    for b in blocks(ins):
        n_mma = sum(1 for x in b if "MMA" in x[1])
        if n_mma >= 8:
            print(f"block @{b[0][0]:05x}: {len(b)} instr, {n_mma} MMA, stall sum {sum(x[2] for x in b)} cycles")
            if "--dump" in sys.argv:
                for x in b:
                    print(f"  {x[0]:05x} s{x[2]:2d} {x[1][:80]}")
