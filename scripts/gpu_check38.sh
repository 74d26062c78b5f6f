# nas-cg + vector-mul: parity tests, C++ GPU tests, device timings
make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -15
timeout 600 ./tests/_bin/vgpu-tests 2>&1 | tail -5
PYTHONPATH=. timeout 600 python scripts/cg_check.py gpurun_out/cg_check.json 2>&1 | tail -12
