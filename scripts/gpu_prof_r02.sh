#!/bin/bash
# ncu --set full capture of the fast kernel of a workload (default cfg3); tag = $2
W=${1:-cfg3}; TAG=${2:-r02}
python scripts/profile_run.py $W 2 > gpurun_out/plain_${W}_${TAG}.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_${W}_${TAG}.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_${W}_${TAG} python scripts/profile_run.py $W 2 > gpurun_out/ncu_${W}_${TAG}.log 2>&1
echo "ncu rc $?"; ls -la gpurun_out/prof_${W}_${TAG}.ncu-rep
