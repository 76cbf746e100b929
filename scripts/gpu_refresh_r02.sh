#!/bin/bash
# round-2 evidence refresh: default bench both arms + cfg2, all workloads, ncu captures
TAG=${1:-r02z}
bash scripts/gpu_bench_r02.sh $TAG
bash scripts/gpu_workloads_r02.sh
bash scripts/gpu_prof_r02.sh cfg3 $TAG
bash scripts/gpu_prof_r02.sh cfg2 $TAG
bash scripts/gpu_prof_calpa.sh $TAG
