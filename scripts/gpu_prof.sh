set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --workload cfg3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
W=${1:-cfg2}
python scripts/profile_run.py $W 2 > gpurun_out/plain_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_${W}_v11 python scripts/profile_run.py $W 2 > gpurun_out/ncu_$W.log 2>&1
