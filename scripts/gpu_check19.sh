make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"; tail -1 gpurun_out/gpu_cpp.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm2_tma -s 3 -c 1 -o gpurun_out/full_mm_tc2 -f ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 2 > gpurun_out/ncu_tc2.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/full_mm_tc2.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/full_mm_tc2.csv 2>&1
timeout 900 python bench.py --workload mm --no-native --no-cpu-baseline --no-kernels > gpurun_out/bench_mm.json 2> gpurun_out/bench_mm.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_mm.json'));print(d['value'], json.dumps(d['roofline']))"
timeout 600 compute-sanitizer --tool memcheck ./paper_1511_07658_b200/bin/payload-bench 0 mm 1 1 2>&1 | grep SUMMARY
timeout 600 compute-sanitizer --tool racecheck ./paper_1511_07658_b200/bin/payload-bench 0 mm 1 1 2>&1 | grep SUMMARY
timeout 600 compute-sanitizer --tool synccheck ./paper_1511_07658_b200/bin/payload-bench 0 mm 1 1 2>&1 | grep SUMMARY
