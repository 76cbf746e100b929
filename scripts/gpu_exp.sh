set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 --workload cfg3 --no-cpu-baseline > gpurun_out/b3.json 2>&1; python scripts/bench_summary.py gpurun_out/b3.json
HDR_LPA_LIB=build/libhdrlpa_o2mb1.so timeout 600 python bench.py --steps 20 --warmup 3 --workload cfg3 --no-cpu-baseline > gpurun_out/b3b.json 2>&1; python scripts/bench_summary.py gpurun_out/b3b.json
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/b2.json 2>&1; python scripts/bench_summary.py gpurun_out/b2.json
