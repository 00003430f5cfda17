#!/usr/bin/env python
"""Per-instruction stall samples of a kernel's hot loop from an ncu report with source import.

  python tools/ncu_loop_stalls.py gpurun_out/x.ncu-rep pipg_fast [min_share] > profiles/rNN_pipg_loop_stalls.txt

The hot loop is taken as the instructions whose execution count equals the most frequent non-zero
count among the most-executed ones (the non-snapshot iteration of the PIPG kernel, the trip of the
power kernel).  Prints the stall-reason totals of the kernel, then the loop in program order with
cumulative sample share; instructions below `min_share` of the loop's samples are folded."""
import collections
import csv
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
min_share = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}


def num(v):
    try:
        return int(v)
    except ValueError:
        return 0


data = [r for r in rows[2:] if len(r) > ix["stall_wait"] and r[ix["Address"]] != "Address"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
total = sum(num(r[ix["# Samples"]]) for r in data)
print(f"# {rows[0][1] if len(rows[0]) > 1 else kernel}")
print(f"# warp-state samples: {total}; share by reason over the whole kernel")
agg = {s: sum(num(r[ix[s]]) for r in data) for s in stalls}
print("#  " + "  ".join(f"{k.replace('stall_', '')} {v / total:.3f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v / total >= 0.005))
counts = collections.Counter(num(r[ix["Instructions Executed"]]) for r in data)
top = sorted((c for c in counts if c > 0), reverse=True)
cands = [c for c in top if counts[c] >= 100]
loop_count = cands[0]
loop = [r for r in data if num(r[ix["Instructions Executed"]]) == loop_count]
ltot = sum(num(r[ix["# Samples"]]) for r in loop)
wf = sum(num(r[ix["L1 Wavefronts Shared"]]) for r in loop)
print(f"# hot loop: {len(loop)} instructions executed {loop_count} times each (per warp: {loop_count} / warps), "
      f"{ltot} samples ({ltot / total:.3f} of the kernel), shared-memory wavefronts per warp-pass {wf / loop_count:.1f}")
mix = collections.Counter()
for r in loop:
    parts = r[ix["Source"]].split()
    op = parts[1] if parts and parts[0].startswith("@") else (parts[0] if parts else "?")
    mix[".".join(op.split(".")[:2]) if op.startswith(("LDS", "STS")) else op.split(".")[0]] += 1
print("# mix: " + "  ".join(f"{k} {v}" for k, v in mix.most_common(14)))
print("# idx  samples  cum   instruction                                                  top stall reasons")
cum = folded = 0
for i, r in enumerate(loop):
    s = num(r[ix["# Samples"]])
    cum += s
    if s / ltot < min_share:
        folded += s
        continue
    tops = sorted(((num(r[ix[k]]), k.replace("stall_", "")) for k in stalls), reverse=True)[:2]
    print(f"{i:5d} {s:7d} {cum / ltot:6.3f}  {r[ix['Source']].strip()[:62]:62s} " + ", ".join(f"{n} {k}" for n, k in tops))
print(f"# {folded} samples ({folded / ltot:.3f}) in instructions below {min_share} each")
