# nas-cg resident placement (all vectors in shared memory, DSMEM pushes)
timeout 1200 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -3
PYTHONPATH=. timeout 600 python scripts/cg_check.py gpurun_out/cg_check9.json 2>&1 | grep -v vmul
for m in 0 1; do echo "mode cap $m"; VGPU_CG_MODE=$m PYTHONPATH=. timeout 600 python scripts/cg_check.py gpurun_out/cg_check9_m$m.json 2>&1 | grep -v vmul | cut -c1-80; done
