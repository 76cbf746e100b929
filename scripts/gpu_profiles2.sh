# Second half of the round profile evidence (kept under gpurun's 64 MiB return limit)
set -x
python -c "import __graft_entry__ as g; g.build()"
python scripts/profile_run.py cfg3 2 > gpurun_out/plain_p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_cfg3_r01 python scripts/profile_run.py cfg3 2 > gpurun_out/ncu_p3.log 2>&1
python scripts/calpa_probe.py > gpurun_out/plain_calpa.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lpa_fast_kernel -s 1 -c 1 -o gpurun_out/prof_calpa_r01 python scripts/calpa_probe.py > gpurun_out/ncu_calpa.log 2>&1
ls -la gpurun_out
