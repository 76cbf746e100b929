# Round profile evidence: bench lines (both arms), the bench launch list and
# one ncu --set full capture per hot kernel (each only after its plain run exits 0)
set -x
R=${1:-r01}
PART=${2:-1}
if [ "$PART" = 1 ]; then
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 python bench.py --workload cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_run.py cfg2 2 > gpurun_out/plain_p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg2_$R python scripts/profile_run.py cfg2 2 > gpurun_out/ncu_p2.log 2>&1
else  # part 2 (gpurun copies back <= 64 MiB per call)
ncu --set full --clock-control none -k regex:"radiance_(phase|merge)_kernel" -s 1 -c 1 -o gpurun_out/prof_cfg2_prepass_$R python scripts/profile_run.py cfg2 2 > gpurun_out/ncu_pp.log 2>&1
python scripts/profile_run.py cfg3 2 > gpurun_out/plain_p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg3_$R python scripts/profile_run.py cfg3 2 > gpurun_out/ncu_p3.log 2>&1
fi
ls -la gpurun_out
