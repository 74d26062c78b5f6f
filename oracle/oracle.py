"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes access to oracle/_build/libvgpu_oracle.so (the C restatements in
vgpu_oracle.c) with numpy helpers. Used by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg as the checker / CPU baseline; never by the
product path (paper_1511_07658_b200/ does not import this module).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB = os.path.join(HERE, "_build", "libvgpu_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")

NPB_VERIFY = {  # NPB 3.x EP verification sums (ep.f), epsilon 1e-8
    24: (-3.247834652034740e3, -6.958407078382297e3),   # class S
    25: (-2.863319731645753e3, -6.320053679109499e3),   # class W
    28: (-4.295875165629892e3, -1.580732573678431e4),   # class A
    30: (4.033815542441498e4, -2.660669192809235e4),    # class B
}


class EpParams(C.Structure):
    _fields_ = [("m", C.c_uint32), ("mk", C.c_uint32), ("first_batch", C.c_uint64),
                ("n_batches", C.c_uint64), ("reserved", C.c_uint64)]


class CgResult(C.Structure):
    _fields_ = [("zeta", C.c_double), ("rnorm", C.c_double), ("niter", C.c_uint32),
                ("n", C.c_uint32), ("nnz", C.c_uint64)]


class MgResult(C.Structure):
    _fields_ = [("rnm2", C.c_double), ("rnmu", C.c_double), ("nx", C.c_uint32),
                ("nit", C.c_uint32), ("reserved", C.c_uint64)]


# NPB 3.x MG classes (mg.f / npbparams): nx (= ny = nz), nit, smoother set,
# published verification value of rnm2 (epsilon 1e-8)
NPB_MG = {
    "S": (32, 4, 0, 0.5307707005734e-04),
    "W": (128, 4, 0, 0.6467329375339e-05),
    "A": (256, 4, 0, 0.2433365309069e-05),
    "B": (256, 20, 1, 0.1800564401355e-05),
}


class EpResult(C.Structure):
    _fields_ = [("q", C.c_uint64 * 10), ("sx", C.c_double), ("sy", C.c_double),
                ("pairs", C.c_uint64), ("n_batches", C.c_uint64)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "oracle"], cwd=REPO, check=True,
                           stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
        L = C.CDLL(LIB)
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        L.vo_vector_add.argtypes = [f32p, f32p, f32p, C.c_size_t]
        L.vo_vector_scale.argtypes = [f32p, f32p, C.c_float, C.c_size_t]
        L.vo_vector_mul.argtypes = [f32p, f32p, f32p, C.c_size_t]
        L.vo_ep_job.argtypes = [C.POINTER(EpParams), C.POINTER(EpResult)]
        L.vo_ep_job.restype = C.c_int
        L.vo_ep_job_lanes.argtypes = [C.POINTER(EpParams), C.POINTER(EpResult)]
        L.vo_ep_job_lanes.restype = C.c_int
        L.vo_ep_log.argtypes = [f64p, f64p, C.c_size_t]
        L.vo_ep_fold.argtypes = [C.POINTER(EpResult), C.c_size_t, C.POINTER(EpResult)]
        L.vo_black_scholes.argtypes = [f32p, f32p, f32p, C.c_size_t, C.c_double, C.c_double,
                                       f64p, f64p]
        L.vo_sgemm.argtypes = [f32p, f32p, C.c_size_t, f64p]
        L.vo_cg_makea.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_void_p,
                                  C.c_uint64]
        L.vo_cg_makea.restype = C.c_uint64
        L.vo_es.argtypes = [C.c_char_p, C.c_uint64, f64p]
        L.vo_es.restype = C.c_int
        L.vo_cg_run.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(CgResult)]
        L.vo_cg_run.restype = C.c_int
        L.vo_mg_make_input.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64]
        L.vo_mg_make_input.restype = C.c_uint64
        L.vo_mg_run.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(MgResult), C.c_void_p]
        L.vo_mg_run.restype = C.c_int
        _lib = L
    return _lib


def vector_add(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    out = np.empty_like(a)
    lib().vo_vector_add(out, a, b, a.size)
    return out


def vector_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    out = np.empty_like(a)
    lib().vo_vector_mul(out, a, b, a.size)
    return out


def vector_scale(x: np.ndarray, f: float) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(x)
    lib().vo_vector_scale(out, x, f, x.size)
    return out


def ep_log(x: np.ndarray) -> np.ndarray:
    """vgpu_ep_log, the EP kernel's shared logarithm, on the CPU."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().vo_ep_log(x, y, x.size)
    return y


def ep_params_bytes(m: int, first: int, count: int, mk: int = 16) -> bytes:
    return bytes(EpParams(m, mk, first, count, 0))


def ep_job(m: int, first: int, count: int, mk: int = 16, lanes: bool = False) -> EpResult:
    """NAS EP job in the kernel's reduction order (lanes=True: the
    lane-sequential order of the branch-free kernel instance)."""
    r = EpResult()
    fn = lib().vo_ep_job_lanes if lanes else lib().vo_ep_job
    rc = fn(C.byref(EpParams(m, mk, first, count, 0)), C.byref(r))
    if rc != 0:
        raise ValueError("bad EP parameters")
    return r


def ep_from_bytes(b: bytes) -> EpResult:
    return EpResult.from_buffer_copy(b)


def ep_fold(parts) -> EpResult:
    arr = (EpResult * len(parts))(*parts)
    out = EpResult()
    lib().vo_ep_fold(arr, len(parts), C.byref(out))
    return out


def black_scholes(S, X, T, r=0.02, v=0.30):
    S, X, T = (np.ascontiguousarray(a, np.float32) for a in (S, X, T))
    call = np.empty(S.size, np.float64)
    put = np.empty(S.size, np.float64)
    lib().vo_black_scholes(S, X, T, S.size, r, v, call, put)
    return call, put


def sgemm(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    n = A.shape[0]
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    Cm = np.empty((n, n), np.float64)
    lib().vo_sgemm(A, B, n, Cm)
    return Cm


# NPB CG classes: (n, nonzer, niter, shift, published zeta) — NPB 3.x cg.f
CG_CLASSES = {
    "S": (1400, 7, 15, 10.0, 8.5971775078648),
    "W": (7000, 8, 15, 12.0, 10.362595087124),
    "A": (14000, 11, 15, 20.0, 17.130235054029),
    "B": (75000, 13, 75, 60.0, 22.712745482631),
    "C": (150000, 15, 75, 110.0, 28.973605592845),
}


def cg_makea(n: int, nonzer: int, niter: int, shift: float) -> bytes:
    need = lib().vo_cg_makea(n, nonzer, niter, shift, None, 0)
    buf = C.create_string_buffer(need)
    lib().vo_cg_makea(n, nonzer, niter, shift, buf, need)
    return buf.raw


def cg_run(inp: bytes) -> "CgResult":
    r = CgResult()
    if lib().vo_cg_run(inp, len(inp), C.byref(r)):
        raise ValueError("malformed nas-cg input")
    return r


def mg_make_input(nx: int, nit: int, coeffs: int) -> bytes:
    """NPB zran3's right-hand side as the nas-mg input (header + nx^3 doubles)."""
    need = lib().vo_mg_make_input(nx, nit, coeffs, None, 0)
    buf = C.create_string_buffer(need)
    lib().vo_mg_make_input(nx, nit, coeffs, buf, need)
    return buf.raw


def mg_run(inp: bytes, with_u: bool = False):
    """The timed part of NPB MG on the CPU: MgResult (and the finest u with
    its ghost layer, (nx+2)^3, when with_u)."""
    r = MgResult()
    nx = int(np.frombuffer(inp[:4], np.uint32)[0])
    u = np.empty((nx + 2) ** 3, np.float64) if with_u else None
    if lib().vo_mg_run(inp, len(inp), C.byref(r), u.ctypes.data if with_u else None):
        raise ValueError("malformed nas-mg input")
    return (r, u) if with_u else r


def mg_from_bytes(b: bytes) -> "MgResult":
    return MgResult.from_buffer_copy(bytes(b[:C.sizeof(MgResult)]))


def cg_from_bytes(b: bytes) -> "CgResult":
    return CgResult.from_buffer_copy(bytes(b[:C.sizeof(CgResult)]))


def es(inp: bytes) -> np.ndarray:
    """binary64 lattice potential [nz, ny, nx] of an electrostatics input."""
    natoms, nx, ny, nz = np.frombuffer(inp[:16], np.uint32)
    out = np.empty(int(nx) * int(ny) * int(nz), np.float64)
    if lib().vo_es(inp, len(inp), out):
        raise ValueError("malformed electrostatics input")
    return out.reshape(int(nz), int(ny), int(nx))


def ref_tool(name: str) -> str:
    """Path of a binary built from the reference sources (oracle/_ref)."""
    return os.path.join(REF_DIR, name)
