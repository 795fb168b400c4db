"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel totals and shares
over the bench's timed sweeps (launches after the last pack_input/pair_gram setup)."""
import collections
import csv
import re
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]  # drop ncu's ==WARNING== lines
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
names = [re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("ifctn::", "") for r in rows]
t = [float(r["Metric Value"]) for r in rows]
# timed region = launches of the last context's sweeps: after the last pack_input
last = max(i for i, n in enumerate(names) if n.startswith("pack_input"))
agg = collections.OrderedDict()
for n, v in zip(names[last + 1:], t[last + 1:]):
    key = re.sub(r"<.*>", lambda m: m.group(0)[:40], n)
    agg.setdefault(key, [0, 0.0])
    agg[key][0] += 1
    agg[key][1] += v
tot = sum(v for _, v in agg.values())
print(f"launches after the last create: {sum(c for c, _ in agg.values())}, total {tot/1e6:.3f} ms (ncu serialised, cold-cache)")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{100*v/tot:6.2f}%  {c:5d} launches  {v/1e6:9.3f} ms  mean {v/c/1e3:9.1f} us  {k}")
