"""3xTF32 tcgen05 SGEMM accuracy at one chunk size (env VGPU_SGEMM_CHUNK):
relative Frobenius error vs binary64 on sampled rows, n in (256, 2048)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07658_b200 import vgpu as V  # noqa: E402

for n in (256, 512, 2048):
    rng = np.random.default_rng(1000)
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    out = V.native_run_task(A.tobytes() + B.tobytes(), V.KernelDescriptor("sgemm"))
    C = np.frombuffer(out, np.float32).reshape(n, n)
    rows = rng.choice(n, 64, replace=False)
    ref = A[rows].astype(np.float64) @ B.astype(np.float64)
    err = np.linalg.norm(C[rows] - ref) / np.linalg.norm(ref)
    print(f"sgemm={os.environ.get('VGPU_SGEMM', 'simt')} chunk={os.environ.get('VGPU_SGEMM_CHUNK', '-')} "
          f"n={n} rel_frob={err:.3e}", flush=True)
