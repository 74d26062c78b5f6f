# round 2 final, part C: after the BS (ftz MUFU) and MG (coarse levels on
# CTA 0) changes: ncu captures of those kernels, the default C3 line, the MG line
mkdir -p gpurun_out/final
O=gpurun_out/final
B=./paper_1511_07658_b200/bin/payload-bench
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_table -s 1 -c 1 -o $O/prof_bs -f $B 0 bs 16 2 > $O/ncu_bs.log 2>&1; echo "ncu bs rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mg_cluster -s 1 -c 1 -o $O/prof_mg2 -f $B 0 mg 8 2 > $O/ncu_mg2.log 2>&1; echo "ncu mg rc=$?"
t0=$(date +%s); timeout 1500 python bench.py > $O/bench_bs2.json 2> $O/bench_bs2.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 1200 python bench.py --workload mg --no-kernels > $O/bench_mg2.json 2> $O/bench_mg2.err; echo "mg rc=$?"
timeout 600 python bench.py --timeline gpurun_out/final/r2_timeline_c3.csv --steps 10 > $O/timeline_c3.json 2>/dev/null; echo "timeline rc=$?"
