#!/usr/bin/env python
"""Per-kernel SASS opcode histogram of libw4a16.so (cuobjdump -sass), for profiles/.

  python tools/sass_hist.py [lib.so] > profiles/r02_sass_opcodes.json

For every kernel: instruction count, the 25 most frequent opcodes (mnemonic without modifiers) and which of
the Blackwell data-path opcodes it contains — UTCHMMA / UTCBAR (tcgen05.mma / commit), STTM / LDTM
(tcgen05.st / ld), UTMALDG (cp.async.bulk.tensor, TMA), UBLKCP (cp.async.bulk), HMMA / IMMA (legacy mma.sync),
LDGSTS (cp.async), LDSM (ldmatrix), SYNCS (mbarrier)."""
import collections
import json
import os
import re
import subprocess
import sys

KEY = ["UTCHMMA", "UTCBAR", "STTM", "LDTM", "UTMALDG", "UBLKCP", "UTMAPF", "HMMA", "IMMA", "LDGSTS", "LDSM", "SYNCS",
       "REDG", "RED", "ATOMG", "MEMBAR", "FENCE"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                             "paper_2505_22179_b200", "libw4a16.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    out, name, ops = {}, None, None

    def close():
        if name is not None:
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            c = collections.Counter(ops)
            out[dem] = {"instructions": len(ops), "top": dict(c.most_common(25)),
                        "blackwell_ops": {k: v for k, v in sorted(c.items()) if any(v2 for v2 in [k in KEY])}}

    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            close()
            name, ops = m.group(1), []
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and ops is not None:
            ops.append(m.group(1))
    close()
    json.dump({"library": os.path.basename(lib), "arch": "sm_100a", "kernels": out}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
