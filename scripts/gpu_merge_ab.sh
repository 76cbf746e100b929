# merged pre-pass mapping A/B: GPU tests on the new build, bench lines, pre-pass launch times
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do for lib in exp/lib_oldmerge.so exp/lib_newmerge.so; do
  HDR_LPA_LIB=$lib timeout 300 python bench.py --steps 50 --warmup 5 --workload cfg2 --no-cpu-baseline > gpurun_out/m_$(basename $lib .so)_$i.json 2>/dev/null
  echo "$lib: $(python scripts/bench_summary.py gpurun_out/m_$(basename $lib .so)_$i.json | cut -c1-100)"
done; done
for lib in exp/lib_oldmerge.so exp/lib_newmerge.so; do
  HDR_LPA_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:radiance_merge -c 20 --csv --log-file gpurun_out/m_ncu_$(basename $lib .so).csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "$lib merge us: $(grep gpu__time gpurun_out/m_ncu_$(basename $lib .so).csv | awk -F'","' '{gsub(/"/,"",$NF); s+=$NF; n++} END {print s/n/1000, n}')"
done
