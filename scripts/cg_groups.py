"""Device timing of nas-cg batches (resident inputs, one launch per step)
with and without group mode: run once per VGPU_CG_GROUPS setting (the
switch is read once per process). Usage: VGPU_CG_GROUPS=1 python scripts/cg_groups.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07658_b200 import vgpu as V  # noqa: E402

res = {}
for cls, k in (("A", 8), ("A", 1), ("W", 8), ("A", 4), ("S", 16)):
    inp = V.cg_input_for_class(cls)
    r = V.resident_bench("nas-cg", [inp] * k, sets=2, warmup=2, steps=4)
    res[f"{cls}x{k}"] = {"ms_per_step": r["ms_per_step"], "jobs_per_s": k / r["ms_per_step"] * 1e3}
    print(cls, k, round(r["ms_per_step"], 3), "ms", flush=True)
print(json.dumps({"groups": os.environ.get("VGPU_CG_GROUPS", "auto"), "join_us": os.environ.get("VGPU_CG_JOIN_US", "50"),
                  "cases": res}))
