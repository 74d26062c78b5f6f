import sys
from paper_1511_07658_b200 import vgpu as V
cls = sys.argv[1] if len(sys.argv) > 1 else "A"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
inp = V.cg_input_for_class(cls, niter=1)
r = V.resident_bench("nas-cg", [inp] * k, sets=1, warmup=1, steps=1)
print(r)
