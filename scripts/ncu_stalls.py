"""Per-stall-reason totals and the top source lines per reason from an ncu
report's source page (usage: ncu_stalls.py report.ncu-rep [n])."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, fname = None, None
tot = collections.Counter()
per = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] in ("Function Name",):
        continue
    if len(r) > 2 and r[2] != "-":  # SASS rows; the "-" rows are the per-line aggregates
        continue
    d = dict(zip(hdr, r))
    key = f"{(fname or "?")[:12]}:{r[0]}"
    src[key] = r[1][:80]
    for k, v in d.items():
        if (k.startswith("stall_") and "Not Issued" not in k) or k == "L2 Theoretical Sectors Local":
            try:
                x = float(v)
            except ValueError:
                continue
            tot[k] += x
            per[k][key] += x
s = sum(v for k, v in tot.items() if k.startswith("stall_"))
for k, v in tot.most_common():
    if k.startswith("stall_"):
        print(f"{k:24s} {v / s * 100:5.1f}%")
print("local-memory L2 sectors", tot["L2 Theoretical Sectors Local"])
for k in ("stall_wait", "stall_short_sb", "stall_branch_resolving", "stall_long_sb",
          "L2 Theoretical Sectors Local"):
    print(f"--- top lines: {k}")
    for key, v in per[k].most_common(n):
        print(f"  {v:12.0f} {key:18s} {src.get(key, '')}")
