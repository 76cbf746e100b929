python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err; echo "bench rc $? $(python scripts/bench_summary.py gpurun_out/bench_final.json | cut -c1-150)"
timeout 300 python bench.py --steps 10 --warmup 3 --workload cfg3 --no-cpu-baseline > gpurun_out/bench_final_cfg3.json 2>/dev/null; echo "cfg3 $(python scripts/bench_summary.py gpurun_out/bench_final_cfg3.json | cut -c1-100)"
