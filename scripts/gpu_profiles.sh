# Round profile evidence: bench lines (both arms), the bench launch list and
# one ncu --set full capture per hot kernel (each only after its plain run exits 0)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_run.py cfg2 2 > gpurun_out/plain_p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg2_r01 python scripts/profile_run.py cfg2 2 > gpurun_out/ncu_p2.log 2>&1
ncu --set full --clock-control none -k regex:"radiance_(phase|merge)_kernel" -s 1 -c 1 -o gpurun_out/prof_cfg2_prepass_r01 python scripts/profile_run.py cfg2 2 > gpurun_out/ncu_pp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lpa_slow_kernel -s 1 -c 1 -o gpurun_out/prof_cfg2_slow_r01 python scripts/profile_run.py cfg2 2 > gpurun_out/ncu_ps.log 2>&1
ls -la gpurun_out
