make -j8 all 2>&1 | tail -1
VGPU_SGEMM=tc2 timeout 60 python scripts/sgemm_tc_check.py; echo "check rc=$?"
VGPU_SGEMM=tc2 timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 10; echo "pb rc=$?"
VGPU_SGEMM=tc timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 10
VGPU_SGEMM=tc2 timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 1 10
nvidia-smi --query-gpu=name,utilization.gpu --format=csv
