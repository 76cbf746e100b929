"""Aggregate ncu stall samples / executed instructions per CUDA source line."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, exe, src = collections.Counter(), collections.Counter(), {}
cur_file = cur = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Function Name", "Line No") or len(r) < 8:
        continue
    if r[0]:
        cur = (cur_file, r[0])
        src[cur] = r[1]
    try:
        agg[cur] += float(r[4] or 0)
        exe[cur] += int(r[7] or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
print("total samples", tot, "warp insts", sum(exe.values()))
for k, v in agg.most_common(n):
    print(f"{v / tot * 100:5.1f}% ex={exe[k]:>10d} {k[0][:12]}:{k[1]:>4s} {src.get(k, '')[:90]}")
