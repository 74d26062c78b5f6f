make -j8 all 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench_ep.json 2> gpurun_out/bench_ep.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_ep.err
python -c "
import json;d=json.load(open('gpurun_out/bench_ep.json'))
print('value',d['value'],'e2e',d['e2e']['value'],'native',d['native']['value'],'ref',d['cpu_baseline']['value'],'ovh',d['overhead_n1']['overhead'],'clk',d['clocks'])
print(json.dumps(d['roofline']))
print(json.dumps(d['kernels']))"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 3 -c 1 -o gpurun_out/full_ep -f ./paper_1511_07658_b200/bin/payload-bench 0 ep 8 2 > gpurun_out/ncu_full_ep.log 2>&1; echo "ncu ep rc=$?"
ncu -i gpurun_out/full_ep.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/full_ep.csv 2>&1
