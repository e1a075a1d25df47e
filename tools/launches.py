"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    per = collections.OrderedDict()
    for r in data:
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else ""
        scale = {"Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6, "msecond": 1e6,
                 "usecond": 1e3, "nsecond": 1.0}.get(unit, 1.0)
        per.setdefault((int(r[ii]), r[ki].split("(")[0][-70:]), {})[r[mi]] = v * scale
    tot = 0.0
    for (i, k), m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        tot += t
        print(f"{i:3d} {k:70s} {t / 1e3:9.1f} us  rd {m.get('dram__bytes_read.sum', 0):8.1f} MB"
              f"  wr {m.get('dram__bytes_write.sum', 0):8.1f} MB")
    print(f"total {tot / 1e6:.3f} ms over {len(per)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
