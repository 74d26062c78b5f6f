# electrostatics: parity tests, device timing, bench line
timeout 900 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -3
PYTHONPATH=. timeout 600 python - <<'PY'
from paper_1511_07658_b200 import workloads as W, vgpu as V
sz = W.Sizes()
for k in (1, 8):
    ins = [W.job_input("es", w, k, sz) for w in range(k)]
    r = V.resident_bench("electrostatics", ins, sets=2, warmup=2, steps=10)
    inter = r["algo_flops_per_launch"] * r["launches_per_step"]
    print(k, "jobs: ms/launch", round(r["kernel_ms_per_launch"], 3), "T rsqrt/s", round(inter / (r["ms_per_step"] * 1e-3) / 1e12, 3), "frac of 148x16x1.965G", round(inter / (r["ms_per_step"] * 1e-3) / (148 * 16 * 1.965e9), 3))
PY
timeout 1200 python bench.py --workload es --steps 10 --warmup 3 --no-kernels > gpurun_out/bench_es.json 2> gpurun_out/bench_es.err; echo "es rc=$?"
tail -2 gpurun_out/bench_es.err | cut -c1-300
python -c "
import json; d=json.load(open('gpurun_out/bench_es.json')); print(d['value'], d['e2e']['value'], d.get('vs_native'), json.dumps(d['roofline'])[:400], d.get('cpu_baseline'))"
