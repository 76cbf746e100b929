"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launches / mean / total / share, for this library's kernels only
(torch's synthetic-frame simulation and the DFMA peak probe excluded)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    # ncu prints the namespace or not depending on the capture mode
    ours = "hdrlpa::" in name or any(
        k in name for k in ("lpa_", "radiance_", "table_copy", "steering_field", "sample_planes",
                            "saturation_mask"))
    if not ours or "fp64_probe" in name:
        continue
    us = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    if unit in ("ns", "nsecond"):
        us /= 1e3
    elif unit in ("ms", "msecond"):
        us *= 1e3
    name = name.split("(")[0]
    rows.append((name, us))
agg = defaultdict(list)
for n, us in rows:
    agg[n].append(us)
tot = sum(us for _, us in rows)
print("kernel, launches, mean_us, total_us, share")
for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{n}, {len(v)}, {sum(v) / len(v):.1f}, {sum(v):.1f}, {sum(v) / tot:.3f}")
