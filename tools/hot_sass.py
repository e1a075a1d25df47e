"""Top stalled SASS lines of one kernel in an ncu report:
   python tools/hot_sass.py report.ncu-rep <kernel-regex> [launch-skip] [n]"""
import csv
import io
import subprocess
import sys


def main(rep, kern, skip="0", n="25"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
    hdr = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]

    def I(x):
        try:
            return int(x)
        except ValueError:
            return 0
    si, src, ie = (hdr.index(c) for c in ("Warp Stall Sampling (All Samples)", "Source", "Instructions Executed"))
    stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(I(r[si]) for r in data)
    print(f"samples {tot}  sass lines {len(data)}  executed {sum(I(r[ie]) for r in data)}")
    agg = {c: sum(I(r[hdr.index(c)]) for r in data) for c in stalls}
    print("stall totals:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:8])
    for r in sorted(data, key=lambda r: -I(r[si]))[: int(n)]:
        top = sorted(((I(r[hdr.index(c)]), c[6:]) for c in stalls if I(r[hdr.index(c)])), reverse=True)[:2]
        print(f"{I(r[si]):6d} {I(r[ie]):9d}  {r[src].strip()[:58]:58s} {top}")


if __name__ == "__main__":
    main(*sys.argv[1:])
