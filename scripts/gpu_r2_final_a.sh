# round 2 final, part A: GPU suite + smoke, default (C3) bench line + its
# reference arm, ncu captures of the changed kernels (EP, MG cluster),
# compute-sanitizer over them
mkdir -p gpurun_out/final
O=gpurun_out/final
B=./paper_1511_07658_b200/bin/payload-bench
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -4 > $O/gputest.txt; tail -2 $O/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
t0=$(date +%s); timeout 1500 python bench.py > $O/bench_bs.json 2> $O/bench_bs.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 900 python bench.py --impl reference > $O/bench_bs_reference_arm.json 2> $O/bench_bs_reference_arm.err; echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 1 -c 1 -o $O/prof_ep -f $B 0 ep 8 2 > $O/ncu_ep.log 2>&1; echo "ncu ep rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mg_cluster -s 1 -c 1 -o $O/prof_mg -f $B 0 mg 8 2 > $O/ncu_mg.log 2>&1; echo "ncu mg rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm2_tma -s 1 -c 1 -o $O/prof_mm -f $B 0 mm 16 2 > $O/ncu_mm.log 2>&1; echo "ncu mm rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool $B 0 ep 1 1 2>&1 | tail -2 | sed "s/^/ep $tool: /"
  timeout 600 compute-sanitizer --tool $tool $B 0 mg 1 1 2>&1 | tail -2 | sed "s/^/mg $tool: /"
done > $O/sanitizer.txt 2>&1; cat $O/sanitizer.txt
timeout 300 $B 0 all > $O/payload_bench.txt 2>&1; echo "payload-bench rc=$?"
