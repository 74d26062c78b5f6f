make -j8 all 2>&1 | tail -1
VGPU_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 --no-native > gpurun_out/tr2.json 2> gpurun_out/tr2.err; echo "torchrun rc=$?"
tail -3 gpurun_out/tr2.err | cut -c1-300
python -c "import json;d=json.load(open('gpurun_out/tr2.json'));print(d['n_gpus'], d['value'], d['e2e']['value'], json.dumps(d['final_reduce']))"
