"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [steps]  > profiles/rNN_launches_summary.txt

Only launches of this repo's kernels (namespace ganq) are counted; the share is of their
summed duration.  Times are ncu's serialised, cold-cache per-launch durations.
"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    if "ganq" not in name:
        continue
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"^void ", "", short)
    short = short.replace("ganq::<unnamed>::", "").replace("ganq::", "")
    unit = r["Metric Unit"]
    v = float(r["Metric Value"].replace(",", ""))
    ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
    rows.append((short, ns))
agg = defaultdict(lambda: [0, 0.0])
for k, ns in rows:
    agg[k][0] += 1
    agg[k][1] += ns
tot = sum(v[1] for v in agg.values())
print(f"# {path}: {len(rows)} launches of ganq kernels, {tot / 1e6:.3f} ms total (ncu, serialised)")
print(f"# per step ({steps} steps): {tot / 1e6 / steps:.3f} ms")
print(f"{'kernel':<48} {'launches':>8} {'ms':>10} {'share':>7} {'us/launch':>10}")
for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:<48} {c:>8} {ns / 1e6:>10.3f} {ns / tot:>7.1%} {ns / c / 1e3:>10.1f}")
