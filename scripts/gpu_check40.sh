# bench lines for the paper's CG and VecMul workloads
make -j8 all 2>&1 | tail -1
timeout 900 python bench.py --workload cg --steps 10 --warmup 3 --no-kernels > gpurun_out/bench_cg.json 2> gpurun_out/bench_cg.err; echo "cg rc=$?"
tail -3 gpurun_out/bench_cg.err | cut -c1-300
timeout 600 python bench.py --workload vmul --steps 20 --warmup 3 --no-kernels > gpurun_out/bench_vmul.json 2> gpurun_out/bench_vmul.err; echo "vmul rc=$?"
tail -3 gpurun_out/bench_vmul.err | cut -c1-300
python - <<'PY'
import json
for w in ("cg", "vmul"):
    try:
        d = json.load(open(f"gpurun_out/bench_{w}.json"))
        print(w, d["value"], d["e2e"]["value"], json.dumps(d.get("vs_native") or d.get("native")), json.dumps({k: d["roofline"].get(k) for k in ("achieved", "frac", "kernel_us_per_launch")}), json.dumps(d.get("cpu_baseline", {}).get("value")))
    except Exception as e:
        print(w, "ERR", e)
PY
