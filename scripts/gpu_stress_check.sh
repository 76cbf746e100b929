# the stress-fuzz cases with razor-edge order-1 decisions + the full GPU suite + perf A/B
HDR_FUZZ_SCALE=30 timeout 900 python -m pytest "tests/test_gpu_fuzz.py::test_random_steered_pass_parity[80]" "tests/test_gpu_fuzz.py::test_random_affine_rig_parity[219]" "tests/test_gpu_fuzz.py::test_random_affine_rig_parity[379]" -q 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
AB_TAG=${AB_TAG:-rf} AB_WL="${AB_WL:-cfg2 cfg3 calpa}" bash scripts/gpu_ab_only.sh
