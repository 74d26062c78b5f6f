# round 2: C++ GPU suite (fault containment retry), 2-rank torchrun bench
# sharing the GPU (test mode) on the default C3 config, 2-daemon launcher run
mkdir -p gpurun_out
nvidia-smi -q | grep -i "compute mode" | head -2
timeout 600 ./tests/_bin/vgpu-tests --only-gpu 2>&1 | tail -4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --no-native --no-cpu-baseline --no-kernels > gpurun_out/r2_bench_bs_torchrun2.json 2> gpurun_out/r2_bench_bs_torchrun2.err; echo "torchrun2 rc=$?"; tail -3 gpurun_out/r2_bench_bs_torchrun2.err; head -c 600 gpurun_out/r2_bench_bs_torchrun2.json; echo
B=paper_1511_07658_b200/bin
timeout 300 $B/vgpu-launch --shared-gpu --gpus 2 --procs-per-gpu 8 --workload ep --rounds 10 --warmup 2 --ep-batches 8192 --ep-m 29 > gpurun_out/r2_launch_ep_2gvm.json 2> gpurun_out/r2_launch_ep_2gvm.err; echo "launch ep rc=$?"; head -c 1200 gpurun_out/r2_launch_ep_2gvm.json; echo; tail -3 gpurun_out/r2_launch_ep_2gvm.err
