timeout 600 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -2
PYTHONPATH=. timeout 300 python scripts/cg_check.py gpurun_out/cg_check12.json 2>&1 | grep -v vmul | cut -c1-90
for m in 2 1 0; do VGPU_CG_GRID=0 VGPU_CG_MODE=$m PYTHONPATH=. timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python scripts/san_one.py cg > gpurun_out/san_rc_cg$m.log 2>&1; echo "racecheck cluster mode $m: $(grep -h SUMMARY gpurun_out/san_rc_cg$m.log | tail -1)"; done
for tool in racecheck memcheck synccheck; do VGPU_CG_GRID=1 PYTHONPATH=. timeout 900 compute-sanitizer --tool $tool --print-limit 3 python scripts/san_one.py cg > gpurun_out/san_${tool}_cggrid.log 2>&1; echo "$tool grid: $(grep -h SUMMARY gpurun_out/san_${tool}_cggrid.log | tail -1)"; done
