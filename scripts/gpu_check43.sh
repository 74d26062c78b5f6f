# full GPU suite + smoke + default bench + reference arm, then nas-cg ncu capture (class A x 8, 1 iteration)
bash scripts/gpu_final.sh
PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_kernel -s 1 -c 1 -o gpurun_out/prof_cg_a8 -f python scripts/cg_one.py A 8 > gpurun_out/ncu_cg8.log 2>&1; echo "ncu cg rc=$?"
