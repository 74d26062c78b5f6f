# FP32 acceptance screen (EP default) vs no screen (VGPU_EP_VARIANT=13)
make -j8 all 2>&1 | tail -1
B=./paper_1511_07658_b200/bin/payload-bench
for r in 1 2 3; do
  echo "== default"; $B 0 ep 8 40 2>&1 | tail -2
  echo "== v13"; VGPU_EP_VARIANT=13 $B 0 ep 8 40 2>&1 | tail -2
done
timeout 900 python -m pytest tests -m gpu -x -q -k "ep" 2>&1 | tail -3
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 1 -c 1 -o gpurun_out/prof_ep_v9 -f $B 0 ep 8 2 > gpurun_out/ncu_ep.log 2>&1; echo "ncu ep rc=$?"
