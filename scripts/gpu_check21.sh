make -j8 all 2>&1 | tail -1
for v in 0 8 9 10; do echo "variant $v"; VGPU_EP_VARIANT=$v timeout 120 python scripts/ep_compact_check.py; VGPU_EP_VARIANT=$v timeout 60 ./paper_1511_07658_b200/bin/payload-bench 0 ep 8 20; done
