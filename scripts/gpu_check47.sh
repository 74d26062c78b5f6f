# nas-cg grid variant (plain co-resident CTAs, global barrier) vs clusters
timeout 300 python -m pytest tests/test_gpu_cg.py -x -q -k "nas_cg" 2>&1 | tail -2
PYTHONPATH=. timeout 300 python scripts/cg_check.py gpurun_out/cg_check11.json 2>&1 | grep -v vmul | cut -c1-90
echo "clusters only (VGPU_CG_GRID=0)"
VGPU_CG_GRID=0 PYTHONPATH=. timeout 300 python scripts/cg_check.py gpurun_out/cg_check11_nogrid.json 2>&1 | grep -v vmul | cut -c1-90
