"""Per-launch table of an ncu --set full report: duration, DRAM bytes, DRAM %/SM %, issue
activity, SM-active spread — and the DRAM traffic mean over the a2 passes (ncu_traffic.json)."""
import csv
import io
import json
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
a2 = []
print(f"{'#':>3} {'kernel':44s} {'us':>8} {'rd MB':>9} {'wr MB':>8} {'dram%':>6} {'sm%':>6} {'issue%':>6} {'act min/avg/max %':>18}")
for i, r in enumerate(rows[2:]):
    d = dict(zip(hdr, r))
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
    f = lambda k: float(d.get(k) or 0)
    us = f("gpu__time_duration.sum") / 1e3          # base unit: ns
    rd = f("dram__bytes_read.sum") / 1e6            # base unit: bytes
    wr = f("dram__bytes_write.sum") / 1e6
    el = f("sm__cycles_elapsed.avg")
    act = [100 * f("sm__cycles_active." + s) / el if el else 0 for s in ("min", "avg", "max")]
    print(f"{i:3d} {name[:44]:44s} {us:8.1f} {rd:9.2f} {wr:8.2f} "
          f"{f('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{f('sm__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{act[0]:5.1f}/{act[1]:5.1f}/{act[2]:5.1f}")
    if "fiber_pass" in name and "2," not in name and "5," not in name:
        a2.append((rd, wr))
n = max(1, len(a2))
print(json.dumps({"a2_launches": len(a2), "a2_dram_bytes_per_launch_mean":
                  round(1e6 * (sum(x for x, _ in a2) + sum(y for _, y in a2)) / n)}))
