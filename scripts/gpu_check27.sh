make -j8 all 2>&1 | tail -1
timeout 60 python scripts/sgemm_tc_check.py; echo "check rc=$?"
timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 10; echo "pb rc=$?"
timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 1 10
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm2 -c 2 --csv ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 2 2>&1 | grep tc_gemm2 | cut -c1-250
