#!/bin/bash
# one iteration: gpu tests (parity) + cfg3 bench (kernel time) [+ extra workloads]
TAG=${1:-it}; shift
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/${TAG}_tests.log
for W in cfg3 "$@"; do
  timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline --no-api-e2e > gpurun_out/${TAG}_$W.json 2>gpurun_out/${TAG}_$W.err
  echo "$W rc $? $(python scripts/bench_summary.py gpurun_out/${TAG}_$W.json | cut -c1-230)"
done
