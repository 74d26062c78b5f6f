# all BASELINE configs through bench.py (round-1 profile refresh)
make -j8 all 2>&1 | tail -1
for w in ep vecadd bs mm mixed; do
  timeout 1500 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['value'], d['e2e']['value'], d.get('vs_native'), (d.get('cpu_baseline') or {}).get('value'), d['roofline']['frac'], (d.get('overhead_n1') or {}).get('overhead'))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ep.csv python bench.py --steps 3 --warmup 3 --no-native --no-cpu-baseline --no-kernels > gpurun_out/ncu_bench_ep.out 2>&1; echo "ncu launches rc=$?"
