"""One device-resident launch of a workload's kernel at bench.py's per-step
shape (for `ncu --set full` captures): python scripts/ncu_one.py cg|es|vmul"""
import sys

from paper_1511_07658_b200 import vgpu as V
from paper_1511_07658_b200 import workloads as W

kind = sys.argv[1]
procs = W.DEFAULT_PROCS[kind]
sz = W.Sizes()
ins = [W.job_input(kind, w, procs, sz) for w in range(procs)]
print(V.resident_bench(W.PAYLOAD[kind], ins, sets=1, warmup=0, steps=1)["ms_per_step"])
