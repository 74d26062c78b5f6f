# round 2: resident-input e2e, 2-daemon launcher run, overhead curve
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
B=paper_1511_07658_b200/bin
timeout 300 $B/vgpu-launch --shared-gpu --gpus 2 --procs-per-gpu 8 --workload ep --rounds 10 --warmup 2 --ep-batches 8192 --ep-m 29 > gpurun_out/r2_launch_ep_2gvm.json 2> gpurun_out/r2_launch_ep_2gvm.err; echo "launch ep rc=$?"; cat gpurun_out/r2_launch_ep_2gvm.json | head -c 1500; echo
timeout 300 $B/vgpu-launch --gpus 1 --procs-per-gpu 16 --workload mixed --rounds 5 --warmup 2 --inplace > gpurun_out/r2_launch_mixed_1gpu.json 2> gpurun_out/r2_launch_mixed_1gpu.err; echo "launch mixed rc=$?"; head -c 1500 gpurun_out/r2_launch_mixed_1gpu.json; echo
timeout 1200 python bench.py > gpurun_out/r2_bench_bs_b.json 2> gpurun_out/r2_bench_bs_b.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_bench_bs_b.err
timeout 900 python bench.py --overhead-curve --steps 10 > gpurun_out/r2_overhead_b.json 2> gpurun_out/r2_overhead_b.err; echo "overhead rc=$?"
