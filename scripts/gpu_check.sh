set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q -s 2>&1 | grep -E "rgb|slow|mism|passed|failed|Error|error" | tail -60
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --workload cfg3 --no-cpu-baseline 2>&1 | tail -3
