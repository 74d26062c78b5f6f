# round 2: GPU tests (MG, model, launcher, APIs) + FIFO copy-queue A/B on C3
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
for f in 1 0; do
  VGPU_COPY_FIFO=$f timeout 900 python bench.py --no-native --no-cpu-baseline --no-kernels --steps 20 > gpurun_out/r2_bench_bs_fifo$f.json 2> gpurun_out/r2_bench_bs_fifo$f.err; echo "fifo=$f rc=$?"
  python - "$f" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/r2_bench_bs_fifo{sys.argv[1]}.json"))
print("fifo", sys.argv[1], "e2e", round(d["e2e"]["value"]), {k: round(v["value"]) for k, v in d["e2e_other_apis"].items()},
      "link", round(d["roofline"]["link"]["achieved"], 1), round(d["roofline"]["link"]["frac"], 3), d["e2e"]["device_stage_us"])
PY
done
