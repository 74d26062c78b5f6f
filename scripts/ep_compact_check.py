"""EP kernel instances (VGPU_EP_VARIANT) vs the oracle in the matching reduction order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_1511_07658_b200 import vgpu as V  # noqa: E402

v = os.environ.get("VGPU_EP_VARIANT")
lanes = v == "11"
for m, first, count in ((24, 0, 256), (28, 512, 512), (28, 0, 4096), (20, 3, 5)):
    got = oracle.ep_from_bytes(V.native_run_task(oracle.ep_params_bytes(m, first, count),
                                                 V.KernelDescriptor("nas-ep")))
    want = oracle.ep_job(m, first, count, lanes=lanes)
    same = bytes(got) == bytes(want)
    print(f"m={m} [{first},+{count}) lanes={lanes} bit-exact={same} sx={got.sx!r} {want.sx!r}",
          flush=True)
