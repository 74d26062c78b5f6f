make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"; tail -1 gpurun_out/gpu_cpp.log
timeout 120 python scripts/ep_compact_check.py; VGPU_EP_VARIANT=11 timeout 120 python scripts/ep_compact_check.py
./paper_1511_07658_b200/bin/payload-bench 0 ep 8 20; ./paper_1511_07658_b200/bin/payload-bench 0 ep 1 10
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 3 -c 1 -o gpurun_out/full_ep -f ./paper_1511_07658_b200/bin/payload-bench 0 ep 8 2 > gpurun_out/ncu_full_ep.log 2>&1; echo "ncu ep rc=$?"
ncu -i gpurun_out/full_ep.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/full_ep.csv 2>&1
