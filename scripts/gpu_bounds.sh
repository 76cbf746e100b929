#!/bin/bash
# memory-safety check without compute-sanitizer (closed on this pool): the GPU
# test-suite and every kernel family (sanitize_run.py) on a -DHDR_DEBUG_BOUNDS=1
# build, whose range checks raise HDR_FAULT_BOUNDS (status() -> RuntimeError)
mkdir -p gpurun_out
HDR_LPA_LIB=exp/lib_dbg.so python scripts/sanitize_run.py all > gpurun_out/bounds_families.log 2>&1; echo "families rc $?"
HDR_LPA_LIB=exp/lib_dbg.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/bounds_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/bounds_tests.log
