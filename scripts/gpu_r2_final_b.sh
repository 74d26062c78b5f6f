# round 2 final, part B: one bench line per other config / paper workload
# (--no-kernels: the kernel table is in the default line), on the final code
mkdir -p gpurun_out/final
O=gpurun_out/final
for w in ep vecadd mm mixed cg es vmul mg; do
  t0=$(date +%s); timeout 1200 python bench.py --workload $w --no-kernels > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$? wall $(( $(date +%s) - t0 )) s"
done
