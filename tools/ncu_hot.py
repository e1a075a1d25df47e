"""Top stalled SASS instructions of one kernel in an .ncu-rep (source page).
usage: python tools/ncu_hot.py <report> <kernel-regex> [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr]
ix = {k: i for i, k in enumerate(h)}
def num(v):
    try:
        return float(v)
    except ValueError:
        return None


data = [r for r in rows[hdr + 1:] if len(r) == len(h) and num(r[ix["Warp Stall Sampling (All Samples)"]]) is not None]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
data.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total samples {tot:.0f}, instructions {len(data)}")
for r in data[:n]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100 * s / max(tot, 1):5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:100]}")
