make -j8 all 2>&1 | tail -1
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"
grep -E "FAIL|minitest|note" gpurun_out/gpu_cpp.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -5
./paper_1511_07658_b200/bin/payload-bench 0 mm 0 10 2>&1
VGPU_SGEMM=simt ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 10 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/prof_tc -f ./paper_1511_07658_b200/bin/payload-bench 0 mm 4 2 > gpurun_out/ncu_tc.log 2>&1; echo "ncu tc rc=$?"
VGPU_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --workload ep --no-native > gpurun_out/b7_tr2.json 2> gpurun_out/b7_tr2.err; echo "torchrun rc=$?"
tail -5 gpurun_out/b7_tr2.err | cut -c1-300; cat gpurun_out/b7_tr2.json | cut -c1-2000
