# new EP log: parity, speed, ncu; N=1 overhead diagnostics
set -x
make -j8 all 2>&1 | tail -1
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"; tail -2 gpurun_out/gpu_cpp.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
B=./paper_1511_07658_b200/bin/payload-bench
$B 0 ep 8 10; $B 0 ep 1 10
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 3 -c 1 -o gpurun_out/full_ep -f $B 0 ep 8 2 > gpurun_out/ncu_full_ep.log 2>&1; echo "ncu ep rc=$?"
ncu -i gpurun_out/full_ep.ncu-rep --page raw --csv --metrics $M > gpurun_out/full_ep.csv 2>&1
for m in 20 28; do
timeout 600 python bench.py --procs 1 --steps 20 --no-cpu-baseline --no-kernels --ep-m $m > gpurun_out/ov_ep$m.json 2> gpurun_out/ov_ep$m.err; echo "ov ep$m rc=$?"
python -c "import json;d=json.load(open('gpurun_out/ov_ep$m.json'));print(json.dumps(d['overhead_n1']));print(d['e2e']['client_stage_us'],d['e2e']['device_stage_us'], d['native']['value'], d['e2e']['value'])"
done
timeout 600 python bench.py --workload vecadd --procs 1 --steps 20 --no-cpu-baseline --no-kernels > gpurun_out/ov_va.json 2> gpurun_out/ov_va.err; echo "ov va rc=$?"
python -c "import json;d=json.load(open('gpurun_out/ov_va.json'));print(json.dumps(d['overhead_n1']));print(d['e2e']['client_stage_us'],d['e2e']['device_stage_us'], d['native']['value'], d['e2e']['value'])"
