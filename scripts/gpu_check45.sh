# racecheck after the entry cluster barrier; full compute-sanitizer table for nas-cg again
for tool in racecheck memcheck synccheck; do
  for m in 2 1 0; do
    VGPU_CG_MODE=$m PYTHONPATH=. timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/san_one.py cg > gpurun_out/san_${tool}_cg$m.log 2>&1
    echo "$tool nas-cg mode $m rc=$? $(grep -h 'SUMMARY' gpurun_out/san_${tool}_cg$m.log | tail -1)"
  done
done
timeout 900 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -2
PYTHONPATH=. timeout 600 python scripts/cg_check.py gpurun_out/cg_check10.json 2>&1 | grep -v vmul | cut -c1-90
