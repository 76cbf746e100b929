"""Print the key fields of bench.py JSON lines (file or stdin)."""
import json
import sys

src = open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin
for line in src:
    line = line.strip()
    if not line.startswith("{"):
        continue
    j = json.loads(line)
    if j.get("impl") == "reference":
        print("reference", j["config"]["workload"], f"{j['value']:.4f} fps", j["cpu_baseline"]["cores"], "cores")
        continue
    r = j["roofline"]
    mpx = f" ({j['mpix_per_s']:.0f} Mpx/s)" if "mpix_per_s" in j else ""
    hbm = f" | hbm frac {r['hbm']['frac']:.4f}" if "hbm" in r else ""
    print(f"{j['config']['workload']}: {j['value']:.1f} fps{mpx} "
          f"e2e {j['e2e']['value']:.1f} fps | kernel {r['kernel_ms']:.3f} ms, {r['bound']} "
          f"{r['achieved']:.2f}/{r['peak']:.2f} {r['unit']} frac {r['frac']:.3f}{hbm} | "
          f"slow {j.get('slow_path_items')} | clocks {j['clocks']} | cpu {j.get('cpu_baseline')}")
