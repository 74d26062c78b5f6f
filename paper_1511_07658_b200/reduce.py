"""The single cross-GPU reduction of a run.

Each GPU's GVM folds its clients' partial records in worker order. The
per-GPU records then cross GPUs in ONE all-gather: NCCL over NVLink through
vgpu_cu_reduce_final, or any all-gather in tests. Every rank folds them in
rank order. Floating-point sums are therefore deterministic: NCCL's own
reduction order is unspecified, so ncclAllReduce is not used.

Record (REC_WIDTH float64): jobs, q[0..9], sx, sy, pairs, n_batches, checksum.
The EP counts stay below 2^53, so float64 carries them exactly.
"""
from __future__ import annotations

import struct
from typing import Iterable, List, Sequence

REC_WIDTH = 16
NPB_EP_VERIFY = {  # NPB 3.x ep.f verification sums (class: m)
    24: (-3.247834652034740e3, -6.958407078382297e3),
    25: (-2.863319731645753e3, -6.320053679109499e3),
    28: (-4.295875165629892e3, -1.580732573678431e4),
    30: (4.033815542441498e4, -2.660669192809235e4),
}


def bits_to_double(h: str) -> float:
    return struct.unpack("<d", int(h, 16).to_bytes(8, "little"))[0]


def empty_record() -> List[float]:
    return [0.0] * REC_WIDTH


def record_from_workers(results: Iterable[dict]) -> List[float]:
    """Fold one GPU's worker results (in worker order) into its record."""
    rec = empty_record()
    for r in sorted(results, key=lambda x: x["worker"]):
        rec[0] += 1.0
        ep = r.get("ep")
        if ep:
            for i in range(10):
                rec[1 + i] += float(ep["q"][i])
            rec[11] = rec[11] + bits_to_double(ep["sx_bits"])
            rec[12] = rec[12] + bits_to_double(ep["sy_bits"])
            rec[13] += float(ep["pairs"])
            rec[14] += float(ep["n_batches"])
        rec[15] = float((int(rec[15]) + int(r["checksum"], 16)) % 1000003)
    return rec


def fold_in_rank_order(flat: Sequence[float], nranks: int) -> List[float]:
    """Fold the all-gathered records (rank-major) in rank order."""
    out = empty_record()
    for r in range(nranks):
        rec = flat[REC_WIDTH * r: REC_WIDTH * (r + 1)]
        for i in range(REC_WIDTH):
            out[i] = out[i] + rec[i]
    out[15] = float(int(out[15]) % 1000003)
    return out


def ep_verdict(rec: Sequence[float], m: int, total: int = 0,
               rank0: Sequence[float] = ()) -> dict:
    """NPB verification of a folded EP record.

    `total` is the number of batches the run's problem has (0: the whole
    class, 2^(m-16)). The folded record is checked against NPB when it
    covers a class NPB publishes sums for (class A at 1 GPU, class B = m 30
    at 4 GPUs under weak scaling). Under weak scaling rank 0's own record
    covers batches [0, 4096), i.e. exactly class A, at every GPU count: it
    is checked as well when given."""
    total = total or 1 << (m - 16)
    covered = int(rec[14])
    out = {"batches": covered, "problem_batches": total, "pairs": int(rec[13]),
           "sx": rec[11], "sy": rec[12]}
    full_class = covered == total == 1 << (m - 16)
    if full_class and m in NPB_EP_VERIFY:
        sxv, syv = NPB_EP_VERIFY[m]
        out["npb_class_m"] = m
        out["npb_rel_err"] = max(abs((rec[11] - sxv) / sxv), abs((rec[12] - syv) / syv))
        out["verified"] = out["npb_rel_err"] < 1e-8
    if rank0 and int(rank0[14]) == 4096 and not (full_class and m == 28):
        sxv, syv = NPB_EP_VERIFY[28]
        err = max(abs((rank0[11] - sxv) / sxv), abs((rank0[12] - syv) / syv))
        out["rank0_class_a_rel_err"] = err
        out["rank0_class_a_verified"] = err < 1e-8
        out["verified"] = out.get("verified", True) and err < 1e-8
    return out
