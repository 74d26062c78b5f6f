make -j8 all 2>&1 | tail -1
VGPU_BENCH_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 5 --warmup 3 --no-native > gpurun_out/tr4.json 2> gpurun_out/tr4.err; echo "torchrun4 rc=$?"
tail -2 gpurun_out/tr4.err | cut -c1-300
python -c "import json;d=json.load(open('gpurun_out/tr4.json'));print(d['n_gpus'], d['value'], d['e2e']['value'], json.dumps(d['final_reduce']))"
