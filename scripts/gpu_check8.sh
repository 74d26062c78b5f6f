# 3xTF32 chunked-drain accuracy / speed sweep
make -j8 all 2>&1 | tail -1
timeout 120 python scripts/sgemm_tc_check.py
for c in 1 2 4 8 64; do
  VGPU_SGEMM=tc VGPU_SGEMM_CHUNK=$c timeout 120 python scripts/sgemm_tc_check.py
  VGPU_SGEMM=tc VGPU_SGEMM_CHUNK=$c ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 10
done
VGPU_SGEMM=tc VGPU_SGEMM_CHUNK=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/full_mm_tc -f ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 2 > gpurun_out/ncu_full_mm_tc.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/full_mm_tc.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/full_mm_tc.csv 2>&1
