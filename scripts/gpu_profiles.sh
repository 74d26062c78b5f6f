./scripts/tune_stream2 > gpurun_out/tune_stream2.txt 2>&1; cat gpurun_out/tune_stream2.txt
# launch list of the default bench command (durations are cold-cache and serialised under ncu)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vecadd.csv python bench.py --steps 3 --warmup 3 --no-native --no-cpu-baseline > gpurun_out/ncu_bench.out 2>&1; echo "ncu launches rc=$?"
wc -l gpurun_out/launches_vecadd.csv
# full captures of each kernel
B=./paper_1511_07658_b200/bin/payload-bench
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 1 -c 1 -o gpurun_out/prof_ep -f $B 0 ep 4 2 > gpurun_out/ncu_ep.log 2>&1; echo "ep rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sgemm128 -s 1 -c 1 -o gpurun_out/prof_mm -f $B 0 mm 4 2 > gpurun_out/ncu_mm.log 2>&1; echo "mm rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_table -s 1 -c 1 -o gpurun_out/prof_bs -f $B 0 bs 4 2 > gpurun_out/ncu_bs.log 2>&1; echo "bs rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:stream_table -s 3 -c 1 -o gpurun_out/prof_vadd -f $B 0 vecadd 4 5 > gpurun_out/ncu_vadd.log 2>&1; echo "vadd rc=$?"
