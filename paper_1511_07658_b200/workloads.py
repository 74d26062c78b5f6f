"""BASELINE.json configs C1-C5 as job lists (mirror of csrc/tools/workloads.hpp).

Used by bench.py's device-resident leg; the SPMD workers (bin/vgpu-spmd)
build the same shapes natively. vecadd and EP inputs are bit-identical to
the workers'; BS/MM values come from numpy (their cost is value-independent).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._native import EpParams

PAYLOAD = {"vecadd": "vector-add", "ep": "nas-ep", "bs": "black-scholes", "mm": "sgemm"}
KINDS = ("vecadd", "ep", "bs", "mm")
DEFAULT_PROCS = {"vecadd": 4, "ep": 8, "bs": 16, "mm": 16, "mixed": 16}
CONFIG_NAME = {
    "vecadd": "C1 vector addition, 1M floats per process",
    "ep": "C2 NAS EP class A split over the processes",
    "bs": "C3 Black-Scholes 4M options per process",
    "mm": "C4 FP32 matrix multiply 2048x2048 per process",
    "mixed": "C5 mixed: workers cycle vecadd/ep/bs/mm",
}


@dataclass
class Sizes:
    vecadd_n: int = 1 << 20
    ep_m: int = 28
    bs_n: int = 4 << 20
    mm_n: int = 2048


def kind_of(workload: str, worker: int) -> str:
    return KINDS[worker % 4] if workload == "mixed" else workload


def ep_slice(workload: str, worker: int, workers: int, sz: Sizes):
    rank, count = (worker // 4, (workers + 2) // 4) if workload == "mixed" else (worker, workers)
    total = 1 << (sz.ep_m - 16)
    per, extra = divmod(total, count)
    first = rank * per + min(rank, extra)
    return first, per + (1 if rank < extra else 0)


def job_input(workload: str, worker: int, workers: int, sz: Sizes = Sizes()) -> bytes:
    k = kind_of(workload, worker)
    if k == "vecadd":
        j = np.arange(sz.vecadd_n)
        a = ((worker + 1) * 1000.0 + (j % 512)).astype(np.float32)
        b = ((j % 512) * 0.25).astype(np.float32)
        return a.tobytes() + b.tobytes()
    if k == "ep":
        first, count = ep_slice(workload, worker, workers, sz)
        return bytes(EpParams(sz.ep_m, 16, first, count, 0))
    rng = np.random.default_rng((5347 if k == "bs" else 1000) + worker)
    if k == "bs":
        n = sz.bs_n
        return (rng.uniform(5, 30, n).astype(np.float32).tobytes()
                + rng.uniform(1, 100, n).astype(np.float32).tobytes()
                + rng.uniform(0.25, 10, n).astype(np.float32).tobytes())
    n = sz.mm_n
    return rng.uniform(-1, 1, 2 * n * n).astype(np.float32).tobytes()


def output_bytes(kind: str, sz: Sizes = Sizes()) -> int:
    return {"vecadd": 4 * sz.vecadd_n, "ep": 112, "bs": 8 * sz.bs_n,
            "mm": 4 * sz.mm_n * sz.mm_n}[kind]


def input_bytes(kind: str, sz: Sizes = Sizes()) -> int:
    return {"vecadd": 8 * sz.vecadd_n, "ep": 32, "bs": 12 * sz.bs_n,
            "mm": 8 * sz.mm_n * sz.mm_n}[kind]


def region_bytes(workload: str, sz: Sizes = Sizes()) -> int:
    kinds = KINDS if workload == "mixed" else (workload,)
    return max(max(input_bytes(k, sz), output_bytes(k, sz)) for k in kinds)
