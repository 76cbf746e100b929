# Parity numbers (printed summaries) + full GPU suite + cfg2/cfg3 bench lines
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -s 2>&1 | grep -E "^\.?[a-z0-9_ ]*\{|rgb|mismatch|slow|passed|failed|Error" > gpurun_out/parity_print.txt
tail -3 gpurun_out/parity_print.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2>gpurun_out/bench_cfg2.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>gpurun_out/bench_cfg3.err
python scripts/bench_summary.py gpurun_out/bench_cfg2.json
python scripts/bench_summary.py gpurun_out/bench_cfg3.json
