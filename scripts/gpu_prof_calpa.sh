#!/bin/bash
# ncu --set full capture of CALPA's steered pass (2nd lpa_fast_kernel launch of frame 1)
TAG=${1:-r02}
python scripts/profile_calpa.py 2 > gpurun_out/plain_calpa_${TAG}.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_calpa_${TAG}.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 3 -c 1 -o gpurun_out/prof_calpa_${TAG} python scripts/profile_calpa.py 2 > gpurun_out/ncu_calpa_${TAG}.log 2>&1
echo "ncu rc $?"; ls -la gpurun_out/prof_calpa_${TAG}.ncu-rep
