# round 2 (re-entry): GPU suite + smoke, peak probes, default (C3) bench line and
# its reference arm, MG line, acceptance 5-7, launch list + ncu captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -rfEs 2>&1 | tail -25 > gpurun_out/r2_gputest.txt; echo "gputest done"; tail -3 gpurun_out/r2_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke.txt
timeout 300 python -c "
from paper_1511_07658_b200 import vgpu as V
import json
print(json.dumps({'fp64_tflops': V.peak_probe('fp64'), 'fp32_tflops': V.peak_probe('fp32'),
                  'link_alloc': V.link_probe(0), 'link_shm': V.link_probe(0, shm=True),
                  'how': 'vgpu_cu_peak_probe: 148x8 CTAs x 256 threads, 8 independent FMA chains per thread, 2 FLOP per FMA, best of 5; vgpu_cu_link_probe: 256 MiB copies x 8, best of 2 after a warm-up'}))" > gpurun_out/r2_peak_probes.json 2>&1; echo "probes rc=$?"
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r2_bench_bs.json 2> gpurun_out/r2_bench_bs.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_bs_reference_arm.json 2> gpurun_out/r2_bench_bs_reference_arm.err; echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 1200 python bench.py --workload mg --no-kernels > gpurun_out/r2_bench_mg.json 2> gpurun_out/r2_bench_mg.err; echo "mg rc=$?"
timeout 1800 python bench.py --acceptance --steps 10 > gpurun_out/r2_acceptance.json 2> gpurun_out/r2_acceptance.err; echo "acceptance rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bs.csv python bench.py --steps 3 --warmup 3 --no-native --no-cpu-baseline --no-kernels > gpurun_out/r2_ncu_bench.out 2>&1; echo "ncu launches rc=$?"
B=./paper_1511_07658_b200/bin/payload-bench
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_table -s 1 -c 1 -o gpurun_out/r2_prof_bs -f $B 0 bs 16 2 > gpurun_out/r2_ncu_bs.log 2>&1; echo "ncu bs rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ep_table -s 1 -c 1 -o gpurun_out/r2_prof_ep -f $B 0 ep 8 2 > gpurun_out/r2_ncu_ep.log 2>&1; echo "ncu ep rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mg_resid -s 8 -c 1 -o gpurun_out/r2_prof_mg -f $B 0 mg 8 2 > gpurun_out/r2_ncu_mg.log 2>&1; echo "ncu mg rc=$?"
timeout 300 $B 0 all > gpurun_out/r2_payload_bench.txt 2>&1; echo "payload-bench rc=$?"
