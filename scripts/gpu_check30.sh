make -j8 all 2>&1 | tail -1
timeout 120 python scripts/ep_compact_check.py
./paper_1511_07658_b200/bin/payload-bench 0 ep 8 20
VGPU_EP_VARIANT=12 ./paper_1511_07658_b200/bin/payload-bench 0 ep 8 20
timeout 600 python -m pytest tests -x -q -m gpu -k "ep or EP or c2" 2>&1 | tail -2
