#!/usr/bin/env python
"""Dynamic instruction mix + stall samples per opcode from `ncu --page source --csv` output.
usage: ncu -i rep --page source --csv --kernel-name regex:K > src.csv; python tools/ncu_source_mix.py src.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si, ei, smp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("# Samples")
wf = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
wfi = hdr.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in hdr else None
mix = collections.defaultdict(lambda: [0, 0, 0, 0])
tot_e = tot_s = 0
for r in rows[2:]:
    if len(r) <= smp:
        continue
    parts = r[si].split()
    op = parts[1] if parts and parts[0].startswith("@") else (parts[0] if parts else "?")
    e, s = int(r[ei] or 0), int(r[smp] or 0)
    m = mix[op]
    m[0] += e
    m[1] += s
    if wf is not None:
        m[2] += int(r[wf] or 0)
        m[3] += int(r[wfi] or 0)
    tot_e += e
    tot_s += s
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total warp-instructions executed {tot_e}, stall samples {tot_s}")
print(f"{'opcode':28s} {'executed':>12s} {'share':>7s} {'samples':>9s} {'share':>7s} {'smem_wavefronts':>16s} {'ideal':>12s}")
for op, m in sorted(mix.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{op:28s} {m[0]:12d} {m[0]/max(tot_e,1):7.3f} {m[1]:9d} {m[1]/max(tot_s,1):7.3f} {m[2]:16d} {m[3]:12d}")
