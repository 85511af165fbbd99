"""Top stall lines of one kernel in an ncu report (source page, SASS view)."""
import csv, subprocess, sys, collections
rep, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-units", "base", "-k", f"regex:{pat}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
def num(x):
    try:
        float(x); return True
    except Exception:
        return False
data = [r for r in rows[2:] if len(r) == len(hdr) and num(r[hdr.index("Warp Stall Sampling (All Samples)")] or "0")]
iss = hdr.index("Warp Stall Sampling (All Samples)"); isrc = hdr.index("Source"); iex = hdr.index("Instructions Executed")
tot = sum(float(r[iss] or 0) for r in data) or 1
print("total samples", tot, "instructions", sum(float(r[iex] or 0) for r in data))
for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:n]:
    print(f"{float(r[iss])/tot*100:5.1f}% ex={r[iex]:>10} {r[isrc][:120]}")
