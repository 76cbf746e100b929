set -x
bash scripts/gpu_ab.sh v32a cfg3 cfg5 cfg4 2>&1 | tail -8
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
