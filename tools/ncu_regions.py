"""Stall samples of an ncu report grouped by the warp-role code regions of
the fused pass (development aid): prints, per contiguous SASS region that
contains samples, the top stall reasons and the hottest instructions.

usage: python tools/ncu_regions.py report.ncu-rep [gap_bytes]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
gap = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x400
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
iall = h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iall] or 0) for r in data)
print(f"total samples {tot:.0f}")
# split into regions at runs of >= gap bytes without samples
regions, cur, last = [], [], None
for r in data:
    a = int(r[ia], 16)
    s = float(r[iall] or 0)
    if s > 0:
        if last is not None and a - last > gap and cur:
            regions.append(cur)
            cur = []
        cur.append(r)
        last = a
if cur:
    regions.append(cur)
for reg in regions:
    t = sum(float(r[iall] or 0) for r in reg)
    if t < 0.01 * tot:
        continue
    c = collections.Counter()
    for r in reg:
        for s in reasons:
            c[s[6:]] += float(r[h.index(s)] or 0)
    ex = max(int(float(r[iex] or 0)) for r in reg)
    print(f"\n{reg[0][ia][-5:]}-{reg[-1][ia][-5:]}  {100 * t / tot:5.1f}%  max exec {ex}  " +
          ", ".join(f"{k}={100 * v / t:.0f}%" for k, v in c.most_common(4)))
    for r in sorted(reg, key=lambda r: -float(r[iall] or 0))[:4]:
        print(f"     {100 * float(r[iall]) / tot:5.1f}%  {r[ia][-5:]}  {r[isrc][:80]}")
