# round-1 re-entry check: build, GPU tests, smoke, default bench, ncu traffic per kernel
set -x
make -j8 all 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"
tail -3 gpurun_out/gpu_cpp.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
./paper_1511_07658_b200/bin/payload-bench 0 all 0 10 > gpurun_out/payload_bench.txt 2>&1; cat gpurun_out/payload_bench.txt
./paper_1511_07658_b200/bin/payload-bench 0 ep 8 10 2>&1
B=./paper_1511_07658_b200/bin/payload-bench
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for spec in "vecadd 4 stream_table" "ep 8 ep_table" "bs 16 bs_table" "mm 16 tc_gemm"; do
  set -- $spec
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o gpurun_out/full_$1 -f $B 0 $1 $2 2 > gpurun_out/ncu_full_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/full_$1.ncu-rep --page raw --csv --metrics $M > gpurun_out/full_$1.csv 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_default.err; cat gpurun_out/bench_default.json | cut -c1-1500
