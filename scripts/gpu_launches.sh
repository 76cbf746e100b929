# launch list of the default bench command (cfg2, 4 lanes), per-launch times under ncu
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:lpa_|radiance_|table_copy" -c 400 --csv --log-file gpurun_out/launches_r01_final.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc $?"
python scripts/launch_summary.py gpurun_out/launches_r01_final.csv | tail -8
