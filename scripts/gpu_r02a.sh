#!/bin/bash
# round 2, first box call: tests, default (cfg3) bench both arms, cfg2 bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r02a_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2>gpurun_out/r02a_bench.err; echo "bench rc $?"; tail -c 600 gpurun_out/r02a_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02a_ref.json 2>gpurun_out/r02a_ref.err; echo "ref rc $?"; tail -c 400 gpurun_out/r02a_ref.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-api-e2e > gpurun_out/r02a_cfg2.json 2>&1; echo "cfg2 rc $?"
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
