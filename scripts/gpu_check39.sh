# nas-cg SpMV with row segments + 4 chains per lane + rowstr in shared memory
timeout 900 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -5
PYTHONPATH=. timeout 600 python scripts/cg_check.py gpurun_out/cg_check6.json 2>&1 | tail -12
