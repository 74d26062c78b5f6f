"""Host link (PCIe) peaks for both host-memory kinds the data plane could
use: cudaHostAlloc'd buffers vs POSIX shm pages registered in place (the
GVM's regions). Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07658_b200 import vgpu as V  # noqa: E402

out = {}
for shm in (False, True):
    for mb in (8, 48, 256):
        out[f"{'shm' if shm else 'alloc'}_{mb}MiB"] = V.link_probe(0, mb << 20, 8, shm=shm)
print(json.dumps(out, indent=1))
