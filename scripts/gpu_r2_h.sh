# round 2: fault containment (C++ child-process case, vgpud respawn), 2-rank torchrun (shared GPU)
mkdir -p gpurun_out
timeout 300 ./tests/_bin/vgpu-tests "fault containment" 2>&1 | tail -5
timeout 300 python -m pytest tests/test_gpu_fault.py -q -x 2>&1 | tail -15
VGPU_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --no-native --no-cpu-baseline --no-kernels > gpurun_out/r2_bench_bs_torchrun2.json 2> gpurun_out/r2_bench_bs_torchrun2.err; echo "torchrun2 rc=$?"; grep -v Warn gpurun_out/r2_bench_bs_torchrun2.err | tail -3; head -c 400 gpurun_out/r2_bench_bs_torchrun2.json; echo
