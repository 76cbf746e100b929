timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for i in 1 2; do for lib in exp/lib_base.so exp/lib_sharp.so; do
  HDR_LPA_LIB=$lib timeout 300 python bench.py --steps 50 --warmup 5 --workload cfg2 --no-cpu-baseline > gpurun_out/exp_$(basename $lib .so)_$i.json 2>/dev/null
  echo "$lib: $(python scripts/bench_summary.py gpurun_out/exp_$(basename $lib .so)_$i.json | cut -c1-140)"
done; done
