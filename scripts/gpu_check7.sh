# control-plane latency after event-polled completions + hot spin
set -x
make -j8 all 2>&1 | tail -1
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"; tail -1 gpurun_out/gpu_cpp.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
nproc; lscpu | grep -E "Model name|NUMA|Socket|Thread|Core"
./paper_1511_07658_b200/bin/payload-bench 0 ep 8 10
for m in 20 28; do
timeout 600 python bench.py --procs 1 --steps 20 --no-cpu-baseline --no-kernels --ep-m $m > gpurun_out/ov_ep$m.json 2> gpurun_out/ov_ep$m.err; echo "ov ep$m rc=$?"
python -c "import json;d=json.load(open('gpurun_out/ov_ep$m.json'));print(json.dumps(d['overhead_n1']));print(d['e2e']['client_stage_us'],d['e2e']['device_stage_us'], d['native']['value'], d['e2e']['value'])"
done
timeout 600 python bench.py --workload vecadd --procs 1 --steps 20 --no-cpu-baseline --no-kernels > gpurun_out/ov_va.json 2> gpurun_out/ov_va.err; echo "ov va rc=$?"
python -c "import json;d=json.load(open('gpurun_out/ov_va.json'));print(json.dumps(d['overhead_n1']));print(d['e2e']['client_stage_us'],d['e2e']['device_stage_us'], d['native']['value'], d['e2e']['value'])"
timeout 1200 python bench.py > gpurun_out/bench_ep.json 2> gpurun_out/bench_ep.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_ep.err; cat gpurun_out/bench_ep.json
