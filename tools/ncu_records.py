"""Refreshes profiles/ncu_metrics.json and profiles/traffic.json (bench.py's
roofline.ncu / roofline.traffic) from ncu --set full reports of the SpMM
kernel, one launch each, and writes the text summary next to them.

    python tools/ncu_records.py TAG KEY=REPORT [KEY=REPORT ...]
    e.g. python tools/ncu_records.py r2f config5:sum=gpurun_out/prof_r2f_c5sum.ncu-rep

KEY is "<workload>:<op>" as bench.py looks it up; the summary goes to
profiles/<TAG>_<workload>_<op>_ncu.txt (tools/ncu_summary.py).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {n: (u[i], v[i]) for i, n in enumerate(h)}


def to_bytes(unit, val):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(val.replace(",", "")) * scale


def to_us(unit, val):
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3}[unit]
    return float(val.replace(",", "")) * scale


def main():
    tag = sys.argv[1]
    metrics_p, traffic_p = os.path.join(PROF, "ncu_metrics.json"), os.path.join(PROF, "traffic.json")
    metrics = json.load(open(metrics_p))
    traffic = json.load(open(traffic_p))
    for arg in sys.argv[2:]:
        key, rep = arg.split("=", 1)
        r = raw(rep)
        rd, wr = to_bytes(*r["dram__bytes_read.sum"]), to_bytes(*r["dram__bytes_write.sum"])
        dur = to_us(*r["gpu__time_duration.sum"])
        pct = float(r["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][1])
        hit = float(r["lts__t_sector_hit_rate.pct"][1])
        summary = f"profiles/{tag}_{key.replace(':', '_')}_ncu.txt"
        with open(os.path.join(ROOT, summary), "w") as f:
            f.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "12"],
                                   capture_output=True, text=True).stdout)
        metrics[key] = {"dram_bytes": int(rd + wr), "duration_us": dur, "dram_throughput_pct": pct,
                        "l2_hit_pct": hit, "dram_GBs": (rd + wr) / (dur * 1e-6) / 1e9,
                        "source": f"{summary} (ncu --set full --clock-control none, one launch, {tag} build, "
                                  "torch-generated input)"}
        traffic[key] = int(rd + wr)
        print(key, metrics[key])
    json.dump(metrics, open(metrics_p, "w"), indent=1)
    json.dump(traffic, open(traffic_p, "w"), indent=1)


if __name__ == "__main__":
    main()
