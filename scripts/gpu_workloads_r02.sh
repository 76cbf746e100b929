#!/bin/bash
# every bench workload once (device + e2e; no CPU baseline), for DESIGN / README tables
for W in cfg1 cfg2 cfg3 cfg4 cfg5 calpa samples; do
  timeout 600 python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/wl_$W.json 2> gpurun_out/wl_$W.err
  echo "$W rc $? $(python scripts/bench_summary.py gpurun_out/wl_$W.json 2>/dev/null | cut -c1-170)"
done
