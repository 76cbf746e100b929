# one iteration: A/B of exp/lib_*.so on the order-2 workloads, then the GPU tests
bash scripts/gpu_ab.sh ${AB_TAG:-ab} ${AB_WL:-cfg3 cfg5 cfg4} 2>&1 | tail -12
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
