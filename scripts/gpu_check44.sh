# compute-sanitizer over nas-cg (every vector placement) and vector-mul
for tool in memcheck racecheck synccheck initcheck; do
  for m in 2 1 0; do
    VGPU_CG_MODE=$m PYTHONPATH=. timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/san_one.py cg > gpurun_out/san_${tool}_cg$m.log 2>&1
    echo "$tool nas-cg mode $m rc=$? $(grep -h 'SUMMARY' gpurun_out/san_${tool}_cg$m.log | tail -1)"
  done
  PYTHONPATH=. timeout 600 compute-sanitizer --tool $tool --print-limit 5 python scripts/san_one.py vmul > gpurun_out/san_${tool}_vmul.log 2>&1
  echo "$tool vector-mul rc=$? $(grep -h 'SUMMARY' gpurun_out/san_${tool}_vmul.log | tail -1)"
done
timeout 900 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -2
