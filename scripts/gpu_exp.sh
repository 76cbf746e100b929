# A/B of experimental library builds (exp/lib_*.so) on one workload: bench lines only
W=${1:-cfg3}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for lib in exp/lib_*.so; do
  HDR_LPA_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/exp_$(basename $lib .so).json 2>/dev/null
  echo "$lib: $(python scripts/bench_summary.py gpurun_out/exp_$(basename $lib .so).json | cut -c1-120)"
done
