"""Per-kernel summary of an `ncu --set full` report (for profiles/):
duration, DRAM bytes and GB/s, SM/memory throughput, occupancy, issue
activity, FMA-pipe activity, registers.

    python tools/ncu_summary.py report.ncu-rep [peak_gbs] > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

M = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
     ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
     ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
     ("launch__registers_per_thread", "regs")]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "ms": 1e3, "us": 1.0, "ns": 1e-3, "MB": 1.0, "GB": 1e3, "KB": 1e-3, "B": 1e-6}


def main(rep, peak="6536.4"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for m, _ in M)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# {rep}  (DRAM MB; GB/s = (rd+wr)/duration; peak {peak} GB/s measured)")
    print(f"{'kernel':44s} " + " ".join(f"{n:>8s}" for _, n in M) + "     GB/s  frac")
    for r in rows[2:]:
        vals = []
        for m, _ in M:
            i = h.index(m)
            v = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            vals.append(v)
        gbs = (vals[1] + vals[2]) / vals[0] * 1e3 if vals[0] else 0.0
        name = r[h.index("Kernel Name")].replace("(anonymous namespace)::", "").split("(")[0][:44]
        print(f"{name:44s} " + " ".join(f"{v:8.1f}" for v in vals) + f" {gbs:8.0f} {gbs / float(peak):5.2f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
