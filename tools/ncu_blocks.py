"""Per-basic-block executed-instruction shares of one kernel in an .ncu-rep.
usage: python tools/ncu_blocks.py <report> <kernel-regex> [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n_show = int(sys.argv[3]) if len(sys.argv) > 3 else 14
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr]
ix = {k: i for i, k in enumerate(h)}
data, seen = [], set()
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    try:
        n = float(r[ix["Instructions Executed"]])
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    if r[ix["Address"]] in seen:
        continue
    seen.add(r[ix["Address"]])
    data.append((int(r[ix["Address"]], 16), n, smp, r[ix["Source"]].strip()))
tot = sum(d[1] for d in data)
tsm = sum(d[2] for d in data)
segs, cur = [], None
for a, n, smp, s in data:
    if cur and abs(cur[1] - n) < 1 and a - cur[3] == 16:
        cur[2] += 1
        cur[3] = a
        cur[4].append(s)
        cur[5] += smp
    else:
        if cur:
            segs.append(cur)
        cur = [a, n, 1, a, [s], smp]
segs.append(cur)
segs.sort(key=lambda x: -x[1] * x[2])
print(f"total warp instructions {tot:.4g}, stall samples {tsm:.0f}")
for sg in segs[:n_show]:
    print(f"{sg[0] & 0xfffff:05x} len={sg[2]:3d} execs={sg[1]:.3g} inst={100 * sg[1] * sg[2] / tot:5.1f}% "
          f"stall={100 * sg[5] / max(tsm, 1):5.1f}%  {sg[4][0][:44]} .. {sg[4][-1][:34]}")
