"""profiles/ncu_summary.json from an ncu launch list (+ optional full report):
per-config DRAM bytes per launch of k_render / k_preprocess and the render's
FMA-pipe activity, read by bench.py for the roofline `traffic` fields.

    python tools/ncu_json.py garden gpurun_out/launches_X.csv [gpurun_out/full.ncu-rep]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parents[1] / "profiles" / "ncu_summary.json"
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    out = {}
    for r in data:
        name = ("k_render" if "k_render<" in r[ki] else "k_preprocess" if "k_preprocess<" in r[ki]
                else "k_preprocess_views" if "k_preprocess_views<" in r[ki] else None)
        if name and r[mi].startswith("dram__bytes"):
            out[name] = out.get(name, 0.0) + float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    return out


def main(config, csv_path, rep=None, batch_csv=None):
    d = json.loads(OUT.read_text()) if OUT.exists() else {}
    b = launches(csv_path)
    e = d.setdefault(config, {})
    e["k_render_dram_bytes"] = b.get("k_render")
    e["k_preprocess_dram_bytes"] = b.get("k_preprocess")
    e["source"] = str(csv_path)
    if batch_csv:   # launch list of one batched step: the stage-1 launch's DRAM bytes
        e["k_preprocess_views_dram_bytes"] = launches(batch_csv).get("k_preprocess_views")
        e["batch_source"] = str(batch_csv)
    if rep:
        ms = ["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
              "gpu__time_duration.sum"]
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name", "regex:k_render",
                              "--metrics", ",".join(ms)], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        val = {m: float(rows[2][rows[0].index(m)].replace(",", "")) for m in ms}
        dur_s = val["gpu__time_duration.sum"] * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(
            rows[1][rows[0].index("gpu__time_duration.sum")], 1e-9)
        e["k_render_fma_pipe"] = val[ms[0]] / 100.0
        e["k_render_issue_active"] = val[ms[1]] / 100.0
        # warp instructions issued per second (peak: 148 SMs x 4 schedulers x 1 / clock)
        e["k_render_warp_inst_per_s"] = val[ms[2]] / dur_s
        pm = ["smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name",
                              "regex:k_preprocess_views", "--metrics", ",".join(pm)],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) > 2:
            e["k_preprocess_views_issue_active"] = float(rows[2][rows[0].index(pm[0])]) / 100.0
            e["k_preprocess_views_fp64_pipe"] = float(rows[2][rows[0].index(pm[1])]) / 100.0
    OUT.write_text(json.dumps(d, indent=1) + "\n")
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
