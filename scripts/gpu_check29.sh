timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 3 -c 1 -o gpurun_out/full_ep -f ./paper_1511_07658_b200/bin/payload-bench 0 ep 8 2 > gpurun_out/ncu_full_ep.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/full_ep.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/full_ep.csv 2>&1
