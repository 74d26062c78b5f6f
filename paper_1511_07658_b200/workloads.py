"""BASELINE.json configs C1-C5 (+ the paper's CG and VecMul) as job lists
(mirror of csrc/tools/workloads.hpp).

Used by bench.py's device-resident leg; the SPMD workers (bin/vgpu-spmd)
build the same shapes natively. vecadd and EP inputs are bit-identical to
the workers'; BS/MM values come from numpy (their cost is value-independent).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._native import EpParams

PAYLOAD = {"vecadd": "vector-add", "ep": "nas-ep", "bs": "black-scholes", "mm": "sgemm",
           "cg": "nas-cg", "vmul": "vector-mul", "es": "electrostatics", "mg": "nas-mg"}
KINDS = ("vecadd", "ep", "bs", "mm")  # the kinds `mixed` cycles through (C5)
DEFAULT_PROCS = {"vecadd": 4, "ep": 8, "bs": 16, "mm": 16, "mixed": 16, "cg": 8, "vmul": 4,
                 "es": 8, "mg": 8}
CONFIG_NAME = {
    "vecadd": "C1 vector addition, 1M floats per process",
    "ep": "C2 NAS EP class A split over the processes",
    "bs": "C3 Black-Scholes 4M options per process",
    "mm": "C4 FP32 matrix multiply 2048x2048 per process",
    "mixed": "C5 mixed: workers cycle vecadd/ep/bs/mm",
    "cg": "NAS CG class A per process (paper workload, not a BASELINE config)",
    "vmul": "VecMul 1M floats per process (paper workload, not a BASELINE config)",
    "es": "Electrostatics 100K atoms x 64x64x25 lattice per process (paper workload, not a BASELINE config)",
    "mg": "NAS MG class S (32^3, 4 V-cycles) per process (paper workload, not a BASELINE config)",
}
MG_NX = {"S": 32, "W": 128, "A": 256, "B": 256, "C": 512}
_mg_cache = {}

# NPB CG shapes (n, nonzer) for the region bound (mirror of workloads.hpp)
CG_SHAPES = {"S": (1400, 7), "W": (7000, 8), "A": (14000, 11), "B": (75000, 13), "C": (150000, 15)}
_cg_cache = {}


@dataclass
class Sizes:
    vecadd_n: int = 1 << 20
    ep_m: int = 28
    ep_batches: int = 0  # batches of the whole run's EP problem; 0 = the class, 2^(ep_m-16)

    @staticmethod
    def for_world(world: int) -> "Sizes":
        """Weak scaling: every GPU keeps one class-A-sized slice (4096 NPB
        batches); the run's problem is the first 4096*world batches of the
        EP sequence with m = 28 + ceil(log2 world) (m = 30, class B, at 4
        GPUs). Rank 0's slice is always exactly class A."""
        s = Sizes()
        if world > 1:
            s.ep_m = 28 + (world - 1).bit_length()
            s.ep_batches = 4096 * world
        return s

    def size_args(self) -> list:
        return ["--vecadd-n", str(self.vecadd_n), "--ep-m", str(self.ep_m),
                "--ep-batches", str(self.ep_batches), "--bs-n", str(self.bs_n),
                "--mm-n", str(self.mm_n), "--cg-class", self.cg_class,
                "--es-atoms", str(self.es_atoms), "--mg-class", self.mg_class]
    bs_n: int = 4 << 20
    mm_n: int = 2048
    cg_class: str = "A"
    mg_class: str = "S"
    es_atoms: int = 100000
    es_lattice: tuple = (64, 64, 25)
    es_h: float = 0.5


# NAS EP class A (m = 28): accepted Gaussian pairs (NPB ep.f; pinned by
# tests/golden/ep_oracle.json and the oracle)
EP_CLASS_A_ACCEPTED = 210832767
EP_ACCEPT_RATE = EP_CLASS_A_ACCEPTED / float(1 << 28)


def ep_fp64_ops(pairs: float, accepted: float) -> float:
    """Algorithmic binary64 FLOPs of the restated NPB EP step
    (paper_1511_07658_b200/csrc/common/ep_math.h), counted as the FP64 peak
    counts them: an FMA = 2, every other +,-,*,/,sqrt = 1:
      every pair      x1 = 2u1 - 1, x2 = 2u2 - 1 (4), t = x1^2 + x2^2 (3)  -> 7
      accepted pair   log t (vgpu_ep_log): 7 FMAs (r = z/c - 1, k ln2_hi +
                      logc_hi, 5 Horner steps) + 2 FMAs (low part) = 18, r^2
                      and the final 2 additions = 3 -> 21; -2 log t, / t,
                      sqrt (3); x1 t2, x2 t2 (2); sx, sy (2)                  -> 28
    The LCG and the log's argument reduction are integer work, not counted.
    (Until the end of round 1 every op counted 1, FMAs included: 7 + 19.)"""
    return 7.0 * pairs + 28.0 * accepted


def kind_of(workload: str, worker: int) -> str:
    return KINDS[worker % 4] if workload == "mixed" else workload


def ep_slice(workload: str, worker: int, workers: int, sz: Sizes):
    rank, count = (worker // 4, (workers + 2) // 4) if workload == "mixed" else (worker, workers)
    total = sz.ep_batches or 1 << (sz.ep_m - 16)
    per, extra = divmod(total, count)
    first = rank * per + min(rank, extra)
    return first, per + (1 if rank < extra else 0)


def cg_input(cls: str) -> bytes:
    """The CG program's matrix (NPB makea through the product's client-side
    builder, vgpu_cg_make_input); the same for every worker, built once."""
    if cls not in _cg_cache:
        from .vgpu import cg_input_for_class
        _cg_cache[cls] = cg_input_for_class(cls)
    return _cg_cache[cls]


def mg_input(cls: str) -> bytes:
    """The MG program's right-hand side (NPB zran3 through the product's
    client-side builder, vgpu_mg_make_input); the same for every worker."""
    if cls not in _mg_cache:
        from .vgpu import mg_input_for_class
        _mg_cache[cls] = mg_input_for_class(cls)
    return _mg_cache[cls]


def mg_workspace_bytes(nx: int) -> int:
    """vgpu_mg_workspace_bytes: u and r on every level plus the norm partials."""
    b, m = 0, 2
    while m <= nx:
        b += 2 * 8 * (m + 2) ** 3
        m *= 2
    return b + 16 * nx + 256


def job_input(workload: str, worker: int, workers: int, sz: Sizes = Sizes()) -> bytes:
    k = kind_of(workload, worker)
    if k == "cg":
        return cg_input(sz.cg_class)
    if k == "mg":
        return mg_input(sz.mg_class)
    if k == "es":
        return es_input_native(worker, sz)
    if k in ("vecadd", "vmul"):
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


def es_input_native(worker: int, sz: Sizes) -> bytes:
    """An ES job of the configured size (numpy values: like BS/MM, the
    kernel's cost does not depend on them)."""
    from .vgpu import es_input
    nx, ny, nz = sz.es_lattice
    h = sz.es_h
    rng = np.random.default_rng(777 + worker)
    n = sz.es_atoms
    at = np.stack([rng.uniform(0, nx * h, n), rng.uniform(0, ny * h, n),
                   rng.uniform(0, nz * h, n), rng.uniform(-1, 1, n)], axis=1).astype(np.float32)
    return es_input(at, nx, ny, nz, h)


def output_bytes(kind: str, sz: Sizes = Sizes()) -> int:
    return {"vecadd": 4 * sz.vecadd_n, "ep": 112, "bs": 8 * sz.bs_n,
            "mm": 4 * sz.mm_n * sz.mm_n, "cg": 32, "mg": 32, "vmul": 4 * sz.vecadd_n,
            "es": 4 * sz.es_lattice[0] * sz.es_lattice[1] * sz.es_lattice[2]}[kind]


def cg_input_bound(cls: str) -> int:
    """nas-cg input bytes upper bound (nnz <= n (nonzer + 1)^2)."""
    n, nz = CG_SHAPES[cls]
    nnz = n * (nz + 1) ** 2
    b = 24 + 4 * (n + 1) + 4 * nnz
    return ((b + 7) & ~7) + 8 * nnz


def input_bytes(kind: str, sz: Sizes = Sizes()) -> int:
    if kind == "cg":
        return cg_input_bound(sz.cg_class)
    if kind == "mg":
        return 16 + 8 * MG_NX[sz.mg_class] ** 3
    return {"vecadd": 8 * sz.vecadd_n, "ep": 32, "bs": 12 * sz.bs_n,
            "mm": 8 * sz.mm_n * sz.mm_n, "vmul": 8 * sz.vecadd_n,
            "es": 32 + 16 * sz.es_atoms}[kind]


def region_bytes(workload: str, sz: Sizes = Sizes(), resident: bool = False) -> int:
    """Per-client region. resident: the input stays in the region after the
    result's bytes (vgpu-spmd --resident places it at the result size
    rounded up to 64 KiB)."""
    kinds = KINDS if workload == "mixed" else (workload,)
    if workload == "mg":  # the slot workspace (2 x region) must hold the grids
        nx = MG_NX[sz.mg_class]
        base = max(input_bytes("mg", sz), (mg_workspace_bytes(nx) + 1) // 2)
        return base + (input_bytes("mg", sz) + 65536 if resident else 0)
    if resident:
        return max(((output_bytes(k, sz) + 65535) & ~65535) + input_bytes(k, sz) for k in kinds)
    return max(max(input_bytes(k, sz), output_bytes(k, sz)) for k in kinds)
