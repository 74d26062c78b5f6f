make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"; tail -1 gpurun_out/gpu_cpp.log
timeout 1200 python bench.py > gpurun_out/bench_ep.json 2> gpurun_out/bench_ep.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_ep.err
python -c "import json;d=json.load(open('gpurun_out/bench_ep.json'));print(d['value'],d['e2e']['value'],d.get('vs_native'));print(json.dumps(d['roofline']));print(json.dumps(d['kernels']));print(json.dumps(d['cpu_baseline']));print(json.dumps(d['overhead_n1'])[:300])"
timeout 900 python bench.py --workload mm > gpurun_out/bench_mm.json 2> gpurun_out/bench_mm.err; echo "bench mm rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_mm.json'));print(d['value'],d['e2e']['value'],d.get('vs_native'));print(json.dumps(d['roofline']));print(json.dumps(d['cpu_baseline']))"
