make -j8 all 2>&1 | tail -1
timeout 60 python scripts/sgemm_tc_check.py; echo "check rc=$?"
timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 10; echo "pb rc=$?"
VGPU_SGEMM_TMA=0 timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 16 10
timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 mm 1 10
