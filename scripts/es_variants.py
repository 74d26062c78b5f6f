"""electrostatics kernel variants (VGPU_ES_VARIANT) at the bench shape:
8 jobs x 100K atoms x 64x64x25, device-resident, and accuracy vs binary64.
The variants (FMA-pipe rsqrt offload, 8 points per thread) were measured
with this script and removed afterwards (electrostatics row);
today every variant number runs the kept kernel."""
import os, subprocess, sys
code = r'''
import numpy as np
from oracle import oracle
from paper_1511_07658_b200 import workloads as W, vgpu as V
sz = W.Sizes()
ins = [W.job_input("es", w, 8, sz) for w in range(8)]
r = V.resident_bench("electrostatics", ins, sets=2, warmup=2, steps=10)
inter = r["algo_flops_per_launch"] * r["launches_per_step"]
small = V.es_input(np.random.default_rng(1).uniform(0, 10, (3000, 4)).astype(np.float32) - np.array([0, 0, 0, 5], np.float32), 40, 20, 4, 0.5)
got = np.frombuffer(V.native_run_task(small, V.KernelDescriptor("electrostatics")), np.float32).astype(np.float64)
ref = oracle.es(small).ravel()
print(round(r["kernel_ms_per_launch"], 3), "ms", round(inter / (r["ms_per_step"] * 1e-3) / (148 * 16 * 1.965e9), 3), "of MUFU", "err %.2e" % (np.abs(got - ref).sum() / np.abs(ref).sum()))
'''
for v in ("0", "1", "2", "3", "4"):
    env = dict(os.environ, PYTHONPATH=".", VGPU_ES_VARIANT=v)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print("variant", v, p.stdout.strip() or p.stderr[-300:], flush=True)
