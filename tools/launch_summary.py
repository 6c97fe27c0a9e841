"""Markdown summary of an ncu launch list (--metrics gpu__time_duration.sum
--csv): every launch in order with its duration, and the per-kernel totals.
  python tools/launch_summary.py gpurun_out/launches_cfg3_pass.csv [title]"""
import csv
import re
import sys
from collections import OrderedDict

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
with open(path) as fp:
    lines = [ln for ln in fp if not ln.startswith("==")]
rows = []
for row in csv.DictReader(lines):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", row["Kernel Name"])
    name = re.sub(r"^void ", "", name).replace("octf::<unnamed>::", "")
    v = float(row["Metric Value"].replace(",", ""))
    us = v / 1000.0 if row["Metric Unit"] == "ns" else v
    rows.append((name, us, row["Grid Size"]))
tot = OrderedDict()
for n, u, _ in rows:
    c, t = tot.get(n, (0, 0.0))
    tot[n] = (c + 1, t + u)
total = sum(u for _, u, _ in rows)
print(f"# {title}\n")
print(f"{len(rows)} launches, {total:.1f} us of kernel time "
      "(ncu per-launch times are cold-cache and serialised)\n")
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for n, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{n[:70]}` | {c} | {t:.1f} | {100 * t / total:.1f} % |")
print("\n## Launches in order\n")
print("| # | kernel | grid | us |\n|---|---|---|---|")
for i, (n, u, g) in enumerate(rows):
    print(f"| {i} | `{n[:70]}` | {g} | {u:.1f} |")
