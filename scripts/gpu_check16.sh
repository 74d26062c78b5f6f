make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"; tail -1 gpurun_out/gpu_cpp.log
./paper_1511_07658_b200/bin/payload-bench 0 ep 8 20; ./paper_1511_07658_b200/bin/payload-bench 0 ep 1 10
