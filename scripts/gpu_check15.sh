make -j8 all 2>&1 | tail -1
for v in 0 6 7 1; do echo "variant $v"; VGPU_EP_VARIANT=$v ./paper_1511_07658_b200/bin/payload-bench 0 ep 8 20; VGPU_EP_VARIANT=$v ./paper_1511_07658_b200/bin/payload-bench 0 ep 1 10; done
