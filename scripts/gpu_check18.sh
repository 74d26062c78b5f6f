make -j8 all 2>&1 | tail -1
VGPU_SGEMM=tc2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm2 -s 3 -c 1 -o gpurun_out/full_mm_tc2 -f ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 2 > gpurun_out/ncu_tc2.log 2>&1; echo "ncu rc=$?"
VGPU_SGEMM=tc2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_ --csv ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 3 2>&1 | grep -E "tc_" | head -12
