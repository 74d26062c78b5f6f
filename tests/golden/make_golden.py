"""Regenerate the committed golden fixtures (run in the build container).

ref_vector_ops.bin  written by oracle/_ref/ref-golden, i.e. by the UNMODIFIED
                    reference library's own vector-add / vector-scale
                    payloads (proj/src/payload.cpp) on mt19937(41) inputs.
ep_oracle.json      the oracle's NAS EP results for classes S, W, A, B with
                    bit patterns (the GPU must match them exactly) next to
                    NPB's published verification sums (the oracle must match
                    those within NPB's epsilon 1e-8).

    make oracle ref && python tests/golden/make_golden.py
"""
import json
import os
import struct
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle  # noqa: E402


def bits(x: float) -> str:
    return struct.pack("<d", x).hex()


def main() -> None:
    subprocess.run([oracle.ref_tool("ref-golden"), HERE], check=True)
    out = {}
    for m in (24, 25, 28, 30):  # classes S, W, A, B
        r = oracle.ep_job(m, 0, 1 << (m - 16))
        sxv, syv = oracle.NPB_VERIFY[m]
        out[str(m)] = {
            "sx": r.sx, "sy": r.sy, "sx_bits": bits(r.sx), "sy_bits": bits(r.sy),
            "q": list(r.q), "pairs": r.pairs,
            "npb_sx": sxv, "npb_sy": syv,
        }
        # class A decomposed over 8 processes (config C2) and folded in order
        if m == 28:
            parts = [oracle.ep_job(28, 512 * p, 512) for p in range(8)]
            f = oracle.ep_fold(parts)
            out["28x8"] = {"sx": f.sx, "sy": f.sy, "sx_bits": bits(f.sx), "sy_bits": bits(f.sy),
                           "q": list(f.q), "pairs": f.pairs,
                           "parts_sx_bits": [bits(p.sx) for p in parts],
                           "parts_sy_bits": [bits(p.sy) for p in parts]}
    with open(os.path.join(HERE, "ep_oracle.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
