set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-700
timeout 600 python bench.py --steps 10 --warmup 3 --workload cfg3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-700
python scripts/profile_run.py cfg2 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg2_v2 python scripts/profile_run.py cfg2 2 > gpurun_out/ncu_cfg2.log 2>&1
python scripts/profile_run.py cfg3 2 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg3_v2 python scripts/profile_run.py cfg3 2 > gpurun_out/ncu_cfg3.log 2>&1
ls gpurun_out
