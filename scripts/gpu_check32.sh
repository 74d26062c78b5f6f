make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 ./tests/_bin/vgpu-tests --only-gpu 2>&1 | tail -1
timeout 600 python bench.py --procs 1 --steps 20 --no-cpu-baseline --no-kernels > gpurun_out/ov_ep28.json 2> gpurun_out/ov_ep28.err; echo "ov rc=$?"
python -c "import json;d=json.load(open('gpurun_out/ov_ep28.json'));print(json.dumps(d['overhead_n1'])[:600])"
