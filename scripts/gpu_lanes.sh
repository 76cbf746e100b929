# default bench (cfg2, 4 lanes, CPU baseline) + lanes 2 vs 4 on the order-2 ICI workloads
timeout 600 python bench.py > gpurun_out/bench_default4.json 2>gpurun_out/bench_default4.err; echo "default: $(python scripts/bench_summary.py gpurun_out/bench_default4.json | cut -c1-140)"
for w in cfg3 cfg5; do for L in 2 4; do
  timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu-baseline --lanes $L > gpurun_out/l_${w}_$L.json 2>/dev/null
  echo "$w lanes $L: $(python scripts/bench_summary.py gpurun_out/l_${w}_$L.json | cut -c1-110)"
done; done
