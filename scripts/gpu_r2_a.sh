# round 2: data-plane change check — GPU tests, default (C3) bench line, overhead curve
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r2_bench_bs_a.json 2> gpurun_out/r2_bench_bs_a.err; echo "bench rc=$?"
tail -5 gpurun_out/r2_bench_bs_a.err
timeout 600 python bench.py --overhead-curve --steps 10 > gpurun_out/r2_overhead_a.json 2> gpurun_out/r2_overhead_a.err; echo "overhead rc=$?"
tail -3 gpurun_out/r2_overhead_a.err
