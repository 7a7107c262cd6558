"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per
kernel (dev tool): python tools/launch_summary.py launches.csv "<command>" """
import csv
import re
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
rd = csv.DictReader(lines)
agg = {}
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    name = re.sub(r"CUB_\d+_SM_\d+::", "", name)
    name = re.sub(r"\(.*$", "", name) if not name.startswith("void") else re.sub(r"\(tcb::EngineArgs.*$|\(.*$", "", name)
    name = name.replace("cub::detail::", "").replace("cub::", "cub::")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
    t, c = agg.get(name[:70], (0.0, 0))
    agg[name[:70]] = (t + ns, c + 1)
tot = sum(t for t, _ in agg.values())
print(f"ncu --metrics gpu__time_duration.sum --clock-control none: {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("(cold-cache, serialised launches; compare shares, not absolutes)\n")
print(f"{'kernel':72s} {'launches':>8s} {'total_ns':>14s} {'share':>7s}")
for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:72s} {c:8d} {t:14.0f} {100 * t / tot:6.2f}%")
