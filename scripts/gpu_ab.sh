#!/bin/bash
# A/B of exp/lib_*.so on workloads (bench lines), optional parity tests with the first lib
TAG=${1:-ab}; shift
for W in "$@"; do
  for lib in exp/lib_*.so; do
    n=$(basename $lib .so)
    HDR_DEBUG_RT=1 HDR_LPA_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline --no-api-e2e > gpurun_out/${TAG}_${n}_$W.json 2>gpurun_out/${TAG}_${n}_$W.err
    echo "$n $W: $(python scripts/bench_summary.py gpurun_out/${TAG}_${n}_$W.json | cut -c1-150) | $(grep -m1 row-tap gpurun_out/${TAG}_${n}_$W.err)"
  done
done
