# Round profile evidence: launch list of the bench command + one full capture per workload
set -x
python -c "import __graft_entry__ as g; g.build()"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_run.py cfg2 2 > gpurun_out/plain_p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg2_r01 python scripts/profile_run.py cfg2 2 > gpurun_out/ncu_p2.log 2>&1
python scripts/profile_run.py cfg3 2 > gpurun_out/plain_p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg3_r01 python scripts/profile_run.py cfg3 2 > gpurun_out/ncu_p3.log 2>&1
ls -la gpurun_out
