"""Summaries of ncu output for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv>   # per-kernel share
  python tools/ncu_summary.py full <report.ncu-rep>      # key counters
"""
import csv
import subprocess
import sys
from collections import defaultdict

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
         "ms": 1e3, "msecond": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    ix = {k: i for i, k in enumerate(rows[h])}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        v = float(r[ix["Metric Value"]].replace(",", ""))
        agg[name][0] += 1
        agg[name][1] += v * SCALE[r[ix["Metric Unit"]]]
    tot = sum(t for _, t in agg.values())
    print("| kernel | launches | total us | avg us | share |")
    print("|---|---:|---:|---:|---:|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:80]}` | {n} | {t:.1f} | {t / n:.1f} | {t / tot * 100:.1f}% |")
    print(f"| total | | {tot:.1f} | | |")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]


def full(path):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"],
                                  text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"kernel: {vals[hdr.index('Kernel Name')][:100]}")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w} = {vals[i]} {units[i]}")


def traffic(path, kernel, workload, out="profiles/r02/ncu_traffic.json"):
    """Append the DRAM bytes per launch of the first kernel in an ncu --set
    full report to ``out``, tagged with the library source hash bench.py
    checks (bench.lib_sha): the bench line cites it only for this build."""
    import json
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"],
                                  text=True)
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                    "Tbyte": 1e12, "ns": 1e-3, "us": 1, "usecond": 1,
                    "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(units[i], 1)
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    rec = {"entries": []}
    if os.path.exists(out):
        rec = json.load(open(out))
    rec["entries"] = [e for e in rec["entries"]
                      if (e["kernel"], e["workload"]) != (kernel, workload)]
    rec["entries"].append({
        "kernel": kernel, "workload": workload, "lib_sha": bench.lib_sha(),
        "kernel_name": vals[hdr.index("Kernel Name")][:120],
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr,
        "duration_us_under_ncu": get("gpu__time_duration.sum"),
        "report": os.path.basename(path)})
    json.dump(rec, open(out, "w"), indent=1)
    print(json.dumps(rec["entries"][-1]))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](
        *sys.argv[2:])
