#!/bin/bash
# round-2 bench evidence: default bench (cfg3) both arms, cfg2 line, ncu launch list of the default command
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc $?"; python scripts/bench_summary.py gpurun_out/${TAG}_bench.json | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc $?"; python scripts/bench_summary.py gpurun_out/${TAG}_ref.json
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err; echo "cfg2 rc $?"; python scripts/bench_summary.py gpurun_out/${TAG}_cfg2.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-api-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc $?"
