# ncu --set full captures of the paper workloads' kernels at bench shape -> DRAM traffic per launch
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for k in cg:cg_kernel es:es_table vmul:stream_table; do
  kind=${k%%:*}; kern=${k##*:}
  PYTHONPATH=. timeout 900 ncu --set full --clock-control none -k regex:$kern -c 1 -o gpurun_out/full_$kind -f python scripts/ncu_one.py $kind > gpurun_out/ncu_$kind.log 2>&1; echo "$kind rc=$?"
  ncu -i gpurun_out/full_$kind.ncu-rep --page raw --csv --metrics $M > gpurun_out/r1_ncu_full_$kind.csv 2>/dev/null
done
