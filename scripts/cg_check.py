"""nas-cg / vector-mul device timings (resident inputs) on cuda:0.

For each NPB class: k jobs in one launch, ms per launch, jobs/s, and the
algorithmic bytes/s (12 B per nonzero per SpMV) against HBM."""
import json
import sys
import time

from paper_1511_07658_b200 import vgpu as V

out = {}
for cls, k in (("S", 1), ("S", 16), ("W", 1), ("W", 8), ("A", 1), ("A", 8)):
    inp = V.cg_input_for_class(cls)
    t0 = time.time()
    r = V.resident_bench("nas-cg", [inp] * k, sets=1, warmup=1, steps=3)
    ms = r["ms_per_step"]
    gbs = r["algo_bytes_per_launch"] * r["launches_per_step"] / (ms * 1e-3) / 1e9
    out[f"{cls}x{k}"] = {"ms_per_step": ms, "jobs_per_s": k / (ms * 1e-3), "launches": r["launches_per_step"],
                        "algo_GBps": gbs, "wall_s": time.time() - t0}
    print(cls, k, json.dumps(out[f"{cls}x{k}"]), flush=True)
for n in (1 << 20, 1 << 22):
    import numpy as np
    a = np.ones(2 * n, np.float32).tobytes()
    r = V.resident_bench("vector-mul", [a] * 4, sets=8, warmup=3, steps=20)
    gbs = r["algo_bytes_per_launch"] / (r["kernel_ms_per_launch"] * 1e-3) / 1e9
    out[f"vmul{n}"] = {"kernel_ms": r["kernel_ms_per_launch"], "GBps": gbs}
    print("vmul", n, json.dumps(out[f"vmul{n}"]), flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cg_check.json", "w"), indent=1)
