# EP headline bench + SIMT sgemm traffic capture + GPU tests
set -x
make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
B=./paper_1511_07658_b200/bin/payload-bench
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sgemm128 -s 3 -c 1 -o gpurun_out/full_mm -f $B 0 mm 16 2 > gpurun_out/ncu_full_mm.log 2>&1; echo "ncu mm rc=$?"
ncu -i gpurun_out/full_mm.ncu-rep --page raw --csv --metrics $M > gpurun_out/full_mm.csv 2>&1
timeout 1200 python bench.py > gpurun_out/bench_ep.json 2> gpurun_out/bench_ep.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_ep.err; cat gpurun_out/bench_ep.json
