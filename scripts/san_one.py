"""One small launch of nas-cg (class S, 2 jobs, 1 outer iteration) or
vector-mul, for compute-sanitizer runs."""
import sys

import numpy as np

from paper_1511_07658_b200 import vgpu as V

if sys.argv[1] == "cg":
    inp = V.cg_input_for_class("S", niter=1)
    print(V.resident_bench("nas-cg", [inp] * 2, sets=1, warmup=0, steps=1)["ms_per_step"])
else:
    a = np.ones(2 * 4099, np.float32).tobytes()
    print(V.resident_bench("vector-mul", [a] * 2, sets=1, warmup=0, steps=1)["ms_per_step"])
