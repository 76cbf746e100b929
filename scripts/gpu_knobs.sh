# cfg2 knobs: exact-path lanes per item (builds) and pipeline lanes (runtime)
for i in 1 2; do
for lib in exp/lib_base.so exp/lib_sl4.so exp/lib_sl16.so; do
  HDR_LPA_LIB=$lib timeout 300 python bench.py --steps 50 --warmup 5 --workload cfg2 --no-cpu-baseline > gpurun_out/k_$(basename $lib .so)_$i.json 2>/dev/null
  echo "$lib: $(python scripts/bench_summary.py gpurun_out/k_$(basename $lib .so)_$i.json | cut -c1-110)"
done
for L in 3 4; do
  timeout 300 python bench.py --steps 50 --warmup 5 --workload cfg2 --no-cpu-baseline --lanes $L > gpurun_out/k_lanes$L_$i.json 2>/dev/null
  echo "lanes $L: $(python scripts/bench_summary.py gpurun_out/k_lanes$L_$i.json | cut -c1-110)"
done; done
