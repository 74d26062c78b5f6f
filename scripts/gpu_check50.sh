# fresh bench lines for C1, C3, C4, C5 on the final code
for w in vecadd bs mm mixed; do
  timeout 1200 python bench.py --workload $w --no-kernels > gpurun_out/bench_${w}_v8.json 2> gpurun_out/bench_${w}_v8.err; echo "$w rc=$?"
done
python - <<'PY'
import json
for w in ("vecadd", "bs", "mm", "mixed"):
    d = json.load(open(f"gpurun_out/bench_{w}_v8.json"))
    r = d["roofline"]
    print(w, round(d["value"]), round(d["e2e"]["value"]), round(d["native"]["value"]), d.get("cpu_baseline", {}).get("value"), r["bound"], round(r["frac"], 3), d["clocks"]["reasons"])
PY
