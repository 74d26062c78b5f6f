# EP kernel occupancy/unroll variants + stream copy effect on vecadd e2e
make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"; tail -1 gpurun_out/gpu_cpp.log
timeout 600 python bench.py --procs 1 --steps 20 --no-cpu-baseline --no-kernels > gpurun_out/ov_ep28.json 2> gpurun_out/ov_ep28.err; echo "ov rc=$?"
python -c "import json;d=json.load(open('gpurun_out/ov_ep28.json'));print(json.dumps(d['overhead_n1'])[:400])"
for v in 0 1 2 3 4 5; do echo "variant $v"; VGPU_EP_VARIANT=$v ./paper_1511_07658_b200/bin/payload-bench 0 ep 8 10; done
timeout 900 python bench.py --workload vecadd --no-native --no-kernels --no-cpu-baseline > gpurun_out/bench_va_nt.json 2> gpurun_out/bench_va_nt.err
VGPU_NO_STREAM_COPY=1 timeout 900 python bench.py --workload vecadd --no-native --no-kernels --no-cpu-baseline > gpurun_out/bench_va_mc.json 2> gpurun_out/bench_va_mc.err
python -c "
import json
for f in ['bench_va_nt','bench_va_mc']:
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['e2e']['value'], d['e2e']['client_stage_us'])"
# launch list of the default bench command (cold-cache, serialised under ncu: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ep.csv python bench.py --steps 3 --warmup 3 --no-native --no-cpu-baseline --no-kernels > gpurun_out/ncu_bench_ep.out 2>&1; echo "ncu launches rc=$?"
wc -l gpurun_out/launches_ep.csv
