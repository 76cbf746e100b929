python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 600 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo bench rc $?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --workload cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>gpurun_out/bench_cfg3.err; echo cfg3 rc $?
