make -j8 all 2>&1 | tail -1
timeout 120 python scripts/ep_compact_check.py
./paper_1511_07658_b200/bin/payload-bench 0 ep 8 20; ./paper_1511_07658_b200/bin/payload-bench 0 ep 1 10
