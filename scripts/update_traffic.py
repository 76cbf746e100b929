"""Regenerate profiles/r02_traffic.json (read by bench.py for the roofline's
`traffic` and the pipe utilisation) from ncu --set full captures.

usage: update_traffic.py workload=gpurun_out/prof_X.ncu-rep[:summary_name] ...
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
path = ROOT / "profiles" / "r02_traffic.json"
data = json.loads(path.read_text()) if path.exists() else {}
for arg in sys.argv[1:]:
    wl, rest = arg.split("=", 1)
    rep, _, summ = rest.partition(":")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    d = dict(zip(rows[0], rows[2]))
    rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
    data[wl] = {
        "kernel": d["Kernel Name"],
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "traffic_bytes": rd + wr,
        "source": f"ncu --set full, profiles/{summ or 'r02_' + wl + '_summary.txt'} ({rep})",
        "fp64_pipe_active_pct": float(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
        "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
        "kernel_ns_ncu": float(d["gpu__time_duration.sum"]),
    }
    print(wl, data[wl]["traffic_bytes"], data[wl]["fp64_pipe_active_pct"])
path.write_text(json.dumps(data, indent=1) + "\n")
