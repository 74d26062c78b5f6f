# compute-sanitizer over every device kernel (small shapes)
make -j8 all 2>&1 | tail -1
B=./paper_1511_07658_b200/bin/payload-bench
for tool in memcheck racecheck synccheck initcheck; do
  for k in vecadd ep bs mm; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 5 $B 0 $k 1 1 > gpurun_out/san_${tool}_$k.log 2>&1
    echo "$tool $k rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' gpurun_out/san_${tool}_$k.log | tail -1)"
  done
done
VGPU_SGEMM=tc timeout 600 compute-sanitizer --tool memcheck $B 0 mm 1 1 2>&1 | grep -E "SUMMARY" | tail -1
VGPU_SGEMM=simt timeout 600 compute-sanitizer --tool memcheck $B 0 mm 1 1 2>&1 | grep -E "SUMMARY" | tail -1
