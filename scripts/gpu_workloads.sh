# bench lines of every workload (no CPU baseline except cfg2's default run)
for w in cfg1 cfg4 cfg5 calpa samples; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err
  echo "$w rc $? $(python scripts/bench_summary.py gpurun_out/bench_$w.json 2>/dev/null | cut -c1-160)"
done
