"""nas-cg class A, one job per launch, at forced cluster widths (VGPU_CG_CLUSTER)."""
import json, os, subprocess, sys
code = r'''
from paper_1511_07658_b200 import vgpu as V
inp = V.cg_input_for_class("A", niter=3)
r = V.resident_bench("nas-cg", [inp], sets=1, warmup=1, steps=3)
print(round(r["ms_per_step"] / (3 * 26) * 1e3, 2))
'''
for cs in (1, 2, 4, 8, 10, 12, 16):
    env = dict(os.environ, PYTHONPATH=".", VGPU_CG_CLUSTER=str(cs))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print("cluster", cs, "us per CG step:", p.stdout.strip() or p.stderr[-300:], flush=True)
