"""nas-cg seg sweep: device ms for classes S x16, W x8, A x1, A x8 (resident)."""
import json, os, subprocess, sys
code = r'''
import json
from paper_1511_07658_b200 import vgpu as V
res = {}
for cls, k in (("S", 16), ("W", 8), ("A", 1), ("A", 8)):
    inp = V.cg_input_for_class(cls)
    r = V.resident_bench("nas-cg", [inp] * k, sets=1, warmup=1, steps=3)
    res[f"{cls}x{k}"] = round(r["ms_per_step"], 3)
print(json.dumps(res))
'''
out = {}
for seg in ("", "8", "16", "32"):
    env = dict(os.environ, PYTHONPATH=".")
    if seg:
        env["VGPU_CG_SEG"] = seg
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    out[seg or "auto"] = p.stdout.strip() or p.stderr[-500:]
    print(seg or "auto", out[seg or "auto"], flush=True)
