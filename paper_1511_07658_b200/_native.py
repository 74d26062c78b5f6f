"""Loader for the in-tree native libraries (ctypes, C-ABI only).

libvgpu_cuda.so  device backend, include/vgpu_cuda.h (nvcc, sm_100a)
libvgpu.so       C++ host stack + include/vgpu_c.h

There is no Python or CPU fallback: if the libraries are missing they are
built with `make` (nvcc + g++ are in the image); if that fails, import fails.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_ROOT = os.path.dirname(PKG_DIR)
LIB_DIR = os.path.join(PKG_DIR, "lib")
BIN_DIR = os.path.join(PKG_DIR, "bin")
LIB_CUDA = os.path.join(LIB_DIR, "libvgpu_cuda.so")
LIB_HOST = os.path.join(LIB_DIR, "libvgpu.so")

_lock = threading.Lock()
_libs = None


def build(target: str = "product", jobs: int = 8) -> None:
    """Compile the native code in-tree (make). Raises on failure."""
    subprocess.run(["make", f"-j{jobs}", target], cwd=REPO_ROOT, check=True,
                   stdout=subprocess.PIPE, stderr=subprocess.STDOUT)


def _artifacts_present() -> bool:
    return all(os.path.exists(p) for p in (LIB_CUDA, LIB_HOST,
                                           os.path.join(BIN_DIR, "vgpu-spmd")))


# ---- C structs -------------------------------------------------------------

class EpParams(C.Structure):
    _fields_ = [("m", C.c_uint32), ("mk", C.c_uint32), ("first_batch", C.c_uint64),
                ("n_batches", C.c_uint64), ("reserved", C.c_uint64)]


class EpResult(C.Structure):
    _fields_ = [("q", C.c_uint64 * 10), ("sx", C.c_double), ("sy", C.c_double),
                ("pairs", C.c_uint64), ("n_batches", C.c_uint64)]


class ResidentResult(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_per_step", C.c_double),
                ("kernel_ms_per_launch", C.c_double), ("launches_per_step", C.c_uint32),
                ("sets", C.c_uint32), ("algo_bytes_per_launch", C.c_uint64),
                ("algo_flops_per_launch", C.c_double), ("resident_bytes", C.c_uint64),
                ("pdl", C.c_uint32), ("reserved", C.c_uint32)]


class LinkResult(C.Structure):
    _fields_ = [("h2d_gbs", C.c_double), ("d2h_gbs", C.c_double), ("bidir_gbs", C.c_double),
                ("bytes", C.c_uint64)]


class CuStats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("tasks", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("batches", C.c_uint64)]


class GvmConfigC(C.Structure):
    _fields_ = [("instance", C.c_char_p), ("max_clients", C.c_uint32),
                ("barrier_size", C.c_uint32), ("per_client_shm_bytes", C.c_uint64),
                ("barrier_window_us", C.c_uint64), ("t_init_us", C.c_uint64),
                ("t_ctx_switch_us", C.c_uint64), ("clock", C.c_int32),
                ("cuda_device", C.c_int32), ("data_plane", C.c_int32),
                ("device_sms", C.c_uint32), ("device_max_kernels", C.c_uint32),
                ("device_slots_per_sm", C.c_uint32), ("scale", C.c_double)]


class DescriptorC(C.Structure):
    _fields_ = [("payload_id", C.c_char_p), ("t_data_in", C.c_uint64), ("t_comp", C.c_uint64),
                ("t_data_out", C.c_uint64), ("grid_size", C.c_uint32),
                ("output_bytes", C.c_uint64)]


class GvmSummary(C.Structure):
    _fields_ = [("tasks", C.c_uint64), ("batches_flushed", C.c_uint64),
                ("uptime_us", C.c_uint64), ("busy_us", C.c_uint64), ("t_init_us", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("device_tasks", C.c_uint64)]


class TaskMetricsC(C.Structure):
    _fields_ = [("task_id", C.c_uint64), ("client_id", C.c_uint32), ("pad", C.c_uint32),
                ("queue_wait_us", C.c_uint64), ("pure_gpu_us", C.c_uint64),
                ("end_to_end_us", C.c_uint64), ("h2d_us", C.c_double),
                ("comp_us", C.c_double), ("d2h_us", C.c_double)]


class BatchMetricsC(C.Structure):
    _fields_ = [("batch_id", C.c_uint64), ("style", C.c_int32), ("task_count", C.c_uint32),
                ("model_makespan_us", C.c_uint64), ("measured_makespan_us", C.c_uint64)]


_P = C.c_void_p
_U32, _U64, _I32, _I64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64

# name -> (restype, argtypes); every function declared in include/vgpu_cuda.h
CUDA_API = {
    "vgpu_cu_open": (C.c_int, [C.c_int, _U32, _U64, C.POINTER(_P)]),
    "vgpu_cu_close": (None, [_P]),
    "vgpu_cu_register_region": (C.c_int, [_P, _U32, _P, _U64]),
    "vgpu_cu_alloc_pinned": (C.c_int, [_P, _U64, C.POINTER(_P)]),
    "vgpu_cu_free_pinned": (None, [_P, _P]),
    "vgpu_cu_payload": (C.c_int, [C.c_char_p, C.POINTER(_U32)]),
    "vgpu_cu_output_size": (C.c_int, [_U32, _P, _U64, C.POINTER(_U64)]),
    "vgpu_cu_task_check": (C.c_int, [_P, _U32, _P, _U64, C.POINTER(_U64)]),
    "vgpu_cu_upload": (C.c_int, [_P, _U32, _P, _U64, _U64]),
    "vgpu_cu_upload_part": (C.c_int, [_P, _U32, _P, _U64, _U64, _U32, _U64]),
    "vgpu_cu_submit_batch": (C.c_int, [_P, C.c_int, _P, _U32, C.POINTER(_U64)]),
    "vgpu_cu_poll": (C.c_int, [_P, _P, _U32, C.POINTER(_U32)]),
    "vgpu_cu_wait": (C.c_int, [_P, _I64]),
    "vgpu_cu_pending": (C.c_int, [_P]),
    "vgpu_cu_get_stats": (C.c_int, [_P, C.POINTER(CuStats)]),
    "vgpu_cu_execute": (C.c_int, [C.c_int, _U32, C.c_float, _P, _U64, _P, _U64, C.POINTER(_U64)]),
    "vgpu_cu_execute_launches": (_U64, []),
    "vgpu_cu_generation": (_U64, [_P]),
    "vgpu_cu_last_fault": (C.c_char_p, [_P]),
    "vgpu_cu_device_lost": (C.c_int, [_P]),
    "vgpu_cu_inject_fault": (C.c_int, [_P, _U32, _U64]),
    "vgpu_cu_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "vgpu_cu_device_pci_bus_id": (C.c_int, [C.c_int, C.c_char_p, C.c_int]),
    "vgpu_cu_task_shape": (C.c_int, [C.c_int, _U32, _P, _U64, C.POINTER(_U32), C.POINTER(_U32)]),
    "vgpu_cu_strerror": (C.c_char_p, [C.c_int]),
    "vgpu_cu_last_error": (C.c_char_p, []),
    "vgpu_cu_resident_bench": (C.c_int, [C.c_int, _U32, C.c_float, _U32, C.POINTER(_P),
                                         C.POINTER(_U64), _U32, _U32, _U32, _U32,
                                         C.POINTER(ResidentResult)]),
    "vgpu_cu_peak_probe": (C.c_int, [C.c_int, _U32, C.POINTER(C.c_double)]),
    "vgpu_cu_launch_probe": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "vgpu_cu_link_probe": (C.c_int, [C.c_int, _U64, _U32, _U32, C.POINTER(LinkResult)]),
    "vgpu_cu_nccl_unique_id": (C.c_int, [_P]),
    "vgpu_cu_comm_init": (C.c_int, [_P, _P, C.c_int, C.c_int]),
    "vgpu_cu_reduce_final": (C.c_int, [_P, _P, _U64, _P]),
}

# every function declared in include/vgpu_c.h
HOST_API = {
    "vgpu_gvm_config_default": (None, [C.POINTER(GvmConfigC)]),
    "vgpu_gvm_start_os": (C.c_int, [C.POINTER(GvmConfigC), C.POINTER(_P)]),
    "vgpu_gvm_stop": (C.c_int, [_P]),
    "vgpu_gvm_destroy": (None, [_P]),
    "vgpu_gvm_summary_get": (C.c_int, [_P, C.POINTER(GvmSummary)]),
    "vgpu_gvm_tasks": (C.c_int, [_P, _P, _U32, C.POINTER(_U32)]),
    "vgpu_gvm_batches": (C.c_int, [_P, _P, _U32, C.POINTER(_U32)]),
    "vgpu_gvm_metrics_csv": (C.c_int, [_P, C.c_char_p, _U64, C.POINTER(_U64)]),
    "vgpu_gvm_timeline_csv": (C.c_int, [_P, C.c_char_p, _U64, C.POINTER(_U64)]),
    "vgpu_unlink_instance": (C.c_int, [C.c_char_p, _U32]),
    "vgpu_gvm_fold": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "vgpu_rendezvous_publish": (C.c_int, [C.c_char_p, _P, _U64]),
    "vgpu_rendezvous_fetch": (C.c_int, [C.c_char_p, _P, _U64, _I64]),
    "vgpu_fold_in_rank_order": (C.c_int, [C.POINTER(C.c_double), _U32, C.POINTER(C.c_double)]),
    "vgpu_local_cpus": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), _U32, C.POINTER(_U32)]),
    "vgpu_client_req": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "vgpu_client_free": (None, [_P]),
    "vgpu_client_id": (_U32, [_P]),
    "vgpu_client_shm_bytes": (_U64, [_P]),
    "vgpu_client_phase": (C.c_int, [_P]),
    "vgpu_client_snd": (C.c_int, [_P, _P, _U64]),
    "vgpu_client_str": (C.c_int, [_P, C.POINTER(DescriptorC)]),
    "vgpu_client_stp": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "vgpu_client_stp_wait": (C.c_int, [_P]),
    "vgpu_client_rcv": (C.c_int, [_P, _P, _U64, C.POINTER(_U64)]),
    "vgpu_client_region": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_U64)]),
    "vgpu_client_snd_region": (C.c_int, [_P, _U64]),
    "vgpu_client_snd_region_at": (C.c_int, [_P, _U64, _U64]),
    "vgpu_client_rcv_region": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_U64)]),
    "vgpu_client_run_task_region": (C.c_int, [_P, _U64, C.POINTER(DescriptorC), C.POINTER(_P),
                                              C.POINTER(_U64)]),
    "vgpu_client_rls": (C.c_int, [_P]),
    "vgpu_client_run_task": (C.c_int, [_P, _P, _U64, C.POINTER(DescriptorC), _P, _U64,
                                       C.POINTER(_U64)]),
    "vgpu_native_run_task": (C.c_int, [C.c_int, C.POINTER(DescriptorC), _P, _U64, _P, _U64,
                                       C.POINTER(_U64)]),
    "vgpu_model_simulate": (_U64, [C.c_int, _U32, _U64, _U64, _U64, _U32, _U32, _U32, _U32]),
    "vgpu_model_simulate_fluid": (_U64, [C.c_int, _U32, _U64, _U64, _U64, _U32, _U32, _U32, _U64, C.c_int]),
    "vgpu_model_classify": (C.c_int, [_U64, _U64, _U64]),
    "vgpu_model_no_vt": (_U64, [_U32, _U64, _U64, _U64, _U64, _U64]),
    "vgpu_encode_frame": (C.c_int, [C.c_uint8, _U32, _U64, _P, _U64, _P, _U64, C.POINTER(_U64)]),
    "vgpu_decode_frame": (C.c_int, [_P, _U64, C.POINTER(C.c_uint8), C.POINTER(_U32),
                                    C.POINTER(_U64), C.POINTER(_U64)]),
    "vgpu_mg_class": (C.c_int, [C.c_char, C.POINTER(_U32), C.POINTER(_U32), C.POINTER(_U32),
                                C.POINTER(C.c_double)]),
    "vgpu_mg_make_input": (C.c_int, [_U32, _U32, _U32, _P, _U64, C.POINTER(_U64)]),
    "vgpu_cg_class": (C.c_int, [C.c_char, C.POINTER(_U32), C.POINTER(_U32), C.POINTER(_U32),
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "vgpu_cg_make_input": (C.c_int, [_U32, _U32, _U32, C.c_double, _P, _U64, C.POINTER(_U64)]),
    "vgpu_last_error": (C.c_char_p, []),
}


class Libs:
    def __init__(self, cuda: C.CDLL, host: C.CDLL):
        self.cuda = cuda
        self.host = host


def _bind(lib: C.CDLL, table: dict) -> None:
    for name, (res, args) in table.items():
        fn = getattr(lib, name)  # AttributeError if the symbol is missing: loud
        fn.restype = res
        fn.argtypes = args


def load(auto_build: bool = True) -> Libs:
    """Load (building first if needed) both libraries; raises if impossible."""
    global _libs
    with _lock:
        if _libs is not None:
            return _libs
        if not _artifacts_present():
            if not auto_build:
                raise OSError("vgpu native libraries are not built (run `make`)")
            build("product")
        mode = getattr(os, "RTLD_GLOBAL", 0) | getattr(os, "RTLD_NOW", 0)
        cuda = C.CDLL(LIB_CUDA, mode=mode)
        host = C.CDLL(LIB_HOST, mode=mode)
        _bind(cuda, CUDA_API)
        _bind(host, HOST_API)
        _libs = Libs(cuda, host)
        return _libs


def bin_path(name: str) -> str:
    return os.path.join(BIN_DIR, name)
