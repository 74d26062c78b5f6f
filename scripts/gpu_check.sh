set -x
make -j8 all 2>&1 | tail -1
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"
grep -E "FAIL|minitest" gpurun_out/gpu_cpp.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
./paper_1511_07658_b200/bin/payload-bench 0 all 0 20 > gpurun_out/payload_bench.txt 2>&1; cat gpurun_out/payload_bench.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:stream_table -s 3 -c 1 -o gpurun_out/prof_vadd -f ./paper_1511_07658_b200/bin/payload-bench 0 vecadd 4 5 > gpurun_out/ncu_vadd.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_vadd.log
